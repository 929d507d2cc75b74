# r02g: fiber kernel (single-chunk staging): parity subset, bench fiber_roofline, ncu pipe metrics
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fiber or wsum or integral or parity_small or smoke" > gpurun_out/r02g_pytest.log 2>&1; tail -2 gpurun_out/r02g_pytest.log
for w in D20 C200; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$w\", round(d['ms_per_step'],3), d['fiber_roofline'])"; done
for w in D20 C200; do
ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__waves_per_multiprocessor --clock-control none -k regex:k_fiber_wsum -c 1 --csv python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02g_ncu_fiber_$w.csv 2>&1
grep -v "^==" gpurun_out/r02g_ncu_fiber_$w.csv | tail -8 | cut -d, -f12-16
done
