# r02g: k_fiber_wsum node-split (cluster) size sweep, D_20 / C_200: average kernel time
for w in D20 C200; do for ns in 1 2 4 8; do
  echo "$w ns=$ns $(TTC_FW_NS=$ns python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["fiber_roofline"]["avg_us"],2), d["integral"]["value"])')"
done; done
