timeout 600 ncu --set full --import-source on --clock-control none -k regex:tsqr_kernel --launch-count 1 -o gpurun_out/tsqr python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_tsqr.log 2>&1; tail -2 gpurun_out/ncu_tsqr.log
ncu -i gpurun_out/tsqr.ncu-rep --page raw --csv > gpurun_out/tsqr_raw.csv 2>/dev/null
ncu -i gpurun_out/tsqr.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/tsqr_lines.csv 2>/dev/null
