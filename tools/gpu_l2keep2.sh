# r02f: L2 evict_last fraction of the TMA factor stream (TTC_L2_KEEP), D_20 / C_200, ms per solve
mkdir -p gpurun_out
for rep in 1 2; do for f in 0 0.1 0.2 0.3 0.45; do for w in D20 C200; do
  echo "$rep $f $w $(TTC_L2_KEEP=$f python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), d["integral"]["value"])')"
done; done; done > gpurun_out/l2keep2.log 2>&1
cat gpurun_out/l2keep2.log
