# k_fiber_wsum cluster-size sweep (TTC_FW_NS) on the large t-form configs
mkdir -p gpurun_out
for ns in 0 1 2 4 8; do for w in D20 C200 C10; do
  echo "$ns $w $(TTC_FW_NS=$ns python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); f=d["fiber_roofline"]; print(d["ms_per_step"], f["avg_us"], f["frac_fp64_peak"])')"
done; done > gpurun_out/fwns.log 2>&1
