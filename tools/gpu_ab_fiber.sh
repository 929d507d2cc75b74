# A/B of library builds on the fiber kernel: "label|ENV|lib" variants, fiber avg_us + solve ms
for rep in 1 2; do for w in ${WLS:-D20 C200}; do for v in $VARIANTS; do
  IFS='|' read -r label envs lib <<< "$v"
  out=$(env $(echo "$envs" | tr "," " ") TTC_LIB_PATH=$PWD/$lib timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["fiber_roofline"]["avg_us"],2), round(d["ms_per_step"],3), d["integral"]["value"])' 2>&1)
  echo "$rep $w $label $out"
done; done; done
