# A/B of two builds on the quadrature fiber kernel time (bench fiber_roofline)
mkdir -p gpurun_out
for rep in 1 2; do for w in D20 C200 D5; do
  for lib in paper_1903_11554_b200/libttcross.so build/libttcross_head.so; do
    echo "$rep $w $lib $(TTC_LIB_PATH=$PWD/$lib python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["fiber_roofline"]["avg_us"])')"
  done
done; done > gpurun_out/abf.log 2>&1
