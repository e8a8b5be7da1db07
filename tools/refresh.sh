#!/bin/bash
# Round-end refresh on one B200 (run under gpurun from the repo root):
# GPU tests, bench lines per config, reference arm, launch lists, traffic,
# full ncu captures of the dominant kernels.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for c in 2 1 3 5 4; do
  timeout 900 python bench.py --config $c > $O/bench_cfg$c.log 2>&1
done
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_cfg2.log 2>&1
bash tools/launch_lists.sh 2 3 5
T=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
timeout 900 ncu -k regex:ozgemm_kernel --metrics $T --clock-control none -c 6 --csv --log-file $O/cfg2_ozgemm_traffic.csv \
  python bench.py --config 2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu -k regex:ozf_kernel --metrics $T --clock-control none -c 4 --csv --log-file $O/cfg5_ozf_traffic.csv \
  python bench.py --config 5 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu -k regex:spmm_kernel --metrics $T --clock-control none -c 12 --csv --log-file $O/cfg3_spmm_traffic.csv \
  python bench.py --config 3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu -k regex:ozgemm_kernel -c 1 --set full --import-source on --clock-control none -o $O/r02_full_ozgemm \
  python bench.py --config 2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
echo done > $O/refresh_done
