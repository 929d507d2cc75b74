mkdir -p gpurun_out
ncu --metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_fiber_wsum -c 1 --csv python bench.py --workload C200 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/fw_flops_c200.csv 2>&1
python bench.py --workload C200 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/c200.json
python bench.py --workload D20 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/d20.json
