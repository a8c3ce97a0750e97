# ncu --set full of the walk7 launch and the seed7 launch of one bench step (config $1, tag $2)
cfg=${1:-5}; tag=${2:-w7}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk7_kernel --launch-count 1 -o gpurun_out/$tag python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1; tail -2 gpurun_out/ncu_$tag.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:seed7_kernel --launch-count 1 -o gpurun_out/${tag}_seed python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${tag}_seed.log 2>&1; tail -2 gpurun_out/ncu_${tag}_seed.log
