# A/B of two builds with the per-phase probe (diagnostics)
mkdir -p gpurun_out
for lib in paper_1903_11554_b200/libttcross.so build/libttcross_head.so; do
  echo "$lib $(TTC_LIB_PATH=$PWD/$lib python bench.py --workload D5 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["integral"]["value"])')"
  TTC_LIB_PATH=$PWD/$lib python tools/probe_phases.py D5 2>&1 | cut -c1-420
done > gpurun_out/abp.log 2>&1
