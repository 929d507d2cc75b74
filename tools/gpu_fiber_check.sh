set -x
mkdir -p gpurun_out
for w in D20 C200 C10 D5; do
  python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/fw_$w.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/fw_pytest.log 2>&1; tail -2 gpurun_out/fw_pytest.log
ncu --set full --clock-control none --import-source on -k regex:k_fiber_wsum -c 1 -o gpurun_out/fw_d20 -f python bench.py --workload D20 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/fw_ncu.log 2>&1
ncu --metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_fiber_wsum -c 3 --csv python bench.py --workload D20 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/fw_flops.csv 2>&1
