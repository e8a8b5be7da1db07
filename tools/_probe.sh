O=gpurun_out
bash tools/launch_lists.sh 1 2 3 5
timeout 600 ncu -k regex:jacobi_rr -c 1 --set full --import-source on --clock-control none -o $O/jac python bench.py --config 2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $O/jac.log 2>&1
ncu -i $O/jac.ncu-rep --page source --csv --print-source=sass > $O/jac_src.csv 2>&1
XB_TRACE=1 timeout 600 python bench.py --config 2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $O/trace2.log 2>&1
