"""Writes tools/xb_kernels.txt: the names of every __global__ function in
paper_1907_06470_b200/csrc (the ncu kernel filter of tools/launch_lists.sh)."""
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    names = set()
    for f in glob.glob(os.path.join(ROOT, "paper_1907_06470_b200", "csrc", "*.cu*")):
        s = open(f).read()
        for m in re.finditer(r"__global__", s):
            t = re.sub(r"__launch_bounds__\s*\([^)]*\)", "", s[m.end():m.end() + 400])
            names.add(re.search(r"([A-Za-z_][A-Za-z_0-9]*)\s*\(", t).group(1))
    with open(os.path.join(ROOT, "tools", "xb_kernels.txt"), "w") as f:
        f.write("|".join(sorted(names)) + "\n")
    print(len(names), "kernels")


if __name__ == "__main__":
    main()
