#!/bin/bash
# ncu launch lists (kernels of libxsvdb200 only) for the given configs
O=gpurun_out
python tools/xb_kernels.py > /dev/null
K="regex:^($(cat tools/xb_kernels.txt | tr -d '\n'))$"
for c in "$@"; do
  timeout 900 ncu --kernel-name-base function -k "$K" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/cfg${c}_launches_xb.csv python bench.py --config $c --steps 1 --warmup 0 \
    --e2e-steps 0 --no-cpu-baseline > $O/cfg${c}_launches_xb.log 2>&1
done
