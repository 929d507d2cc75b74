# L2 evict_last fraction of the rook-step factor stream (TTC_L2_KEEP) on the streaming configs
mkdir -p gpurun_out
for f in 0 0.15 0.25 0.35 0.5; do for w in D20 C200; do
  echo "$f $w $(TTC_L2_KEEP=$f python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["integral"]["value"])')"
done; done > gpurun_out/l2keep.log 2>&1
