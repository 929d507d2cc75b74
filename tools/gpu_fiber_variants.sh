# fiber-kernel variants (build/libttcross_*.so via TTC_LIB_PATH) on the large t-form configs
mkdir -p gpurun_out
for lib in paper_1903_11554_b200/libttcross.so build/libttcross_*.so; do
  for w in D20 C200 D5; do
    echo "$lib $w $(TTC_LIB_PATH=$PWD/$lib python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); f=d["fiber_roofline"]; print(d["ms_per_step"], f["avg_us"], f["frac_fp64_peak"])')"
  done
done > gpurun_out/fv.log 2>&1
