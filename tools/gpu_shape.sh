# k_sweeps launch-shape sweep (TTC_GREEDY_G) on the latency-bound configs
mkdir -p gpurun_out
for g in 16 8 4; do for w in D5 C10 C4; do
  echo "$g $w $(TTC_GREEDY_G=$g python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["launch_shape"])')"
done; done > gpurun_out/shape.log 2>&1
