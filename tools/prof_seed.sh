tag=${1:-seed}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:seed_kernel --launch-count 1 -o gpurun_out/$tag python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1; tail -2 gpurun_out/ncu_$tag.log
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_lines.csv 2>/dev/null
