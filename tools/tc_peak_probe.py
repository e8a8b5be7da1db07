"""tcgen05 peak microbenchmark with constant and with random operand bytes
(power-limited clock): python tools/tc_peak_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_06470_b200 import _lib  # noqa: E402

ctx = _lib.load(0)
for i in range(2):
    print("constant operands: i8 %.0f TOP/s, bf16 %.0f TFLOP/s" % ctx.tc_peaks(), flush=True)
    print("random operands:   i8 %.0f TOP/s, bf16 %.0f TFLOP/s" % ctx.tc_peaks_data(True), flush=True)
