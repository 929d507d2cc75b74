# k_sweeps launch-shape experiments on the full-size configs: cluster size, threads, ring KB
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/shape2.log
for w in D20 C200; do for v in "base|" "g6t512k192|TTC_GREEDY_T=512 TTC_GREEDY_G=6 TTC_RING_KB=192" \
  "g5t512k192|TTC_GREEDY_T=512 TTC_GREEDY_G=5 TTC_RING_KB=192" "g4t512k192|TTC_GREEDY_T=512 TTC_GREEDY_G=4 TTC_RING_KB=192" \
  "g7t512k192|TTC_GREEDY_T=512 TTC_GREEDY_G=7 TTC_RING_KB=192" "g6t512k128|TTC_GREEDY_T=512 TTC_GREEDY_G=6 TTC_RING_KB=128"; do
  IFS='|' read -r label envs <<< "$v"
  out=$(env $envs timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), d["integral"]["value"], round(d["roofline"].get("frac") or 0,4), d["launch_shape"])' 2>&1)
  echo "$w $label $out"
done; done >> gpurun_out/shape2.log 2>&1
cat gpurun_out/shape2.log
