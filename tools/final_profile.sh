# round-end evidence (tag $1): bench lines (cfg5 default, cfg4), the kernel launch list of a
# bench run, ncu --set full of one step's walk launch and seed launch, the walk's FP64
# instruction counts (achieved FP64 FLOP/s)
tag=${1:-rNN}
timeout 600 python bench.py > gpurun_out/${tag}_bench5.json 2> gpurun_out/${tag}_bench5.err; tail -2 gpurun_out/${tag}_bench5.err
timeout 300 python bench.py --config 4 --cpu-seconds 5 > gpurun_out/${tag}_bench4.json 2> gpurun_out/${tag}_bench4.err; tail -2 gpurun_out/${tag}_bench4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/${tag}_ncu_launches.log 2>&1; tail -2 gpurun_out/${tag}_ncu_launches.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_kernel --launch-count 1 -o gpurun_out/${tag}_walk python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_full.log 2>&1; tail -2 gpurun_out/${tag}_ncu_full.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:seed_kernel --launch-count 1 -o gpurun_out/${tag}_seed python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_seed.log 2>&1; tail -2 gpurun_out/${tag}_ncu_seed.log
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:walk_kernel --launch-count 1 --csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_fp64.csv 2> gpurun_out/${tag}_fp64.err; tail -1 gpurun_out/${tag}_fp64.err
