# ring size per SM (L1 carve-out trade-off) and stage shape, r02c
mkdir -p gpurun_out
out=gpurun_out/shape4.log; : > $out
run() {  # workload label envs...
  w=$1; label=$2; shift 2
  r=$(env "$@" timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), d["integral"]["value"], round(d["roofline"].get("frac") or 0,4), d["launch_shape"])' 2>&1 | tail -1)
  echo "$w $label $r" >> $out
}
for rep in 1 2; do
run D20 auto X=1
for kb in 64 96 112 144 160; do run D20 t512g6k$kb TTC_GREEDY_T=512 TTC_GREEDY_G=6 TTC_RING_KB=$kb; done
run D20 t512g6k128tb8 TTC_GREEDY_T=512 TTC_GREEDY_G=6 TTC_RING_KB=128 TTC_RING_TB=8
run D20 t512g6k96tb12 TTC_GREEDY_T=512 TTC_GREEDY_G=6 TTC_RING_KB=96 TTC_RING_TB=12
run D20 t256g6k128 TTC_GREEDY_T=256 TTC_GREEDY_G=6 TTC_RING_KB=128
run D20 t512g7k128 TTC_GREEDY_T=512 TTC_GREEDY_G=7 TTC_RING_KB=128
run C10 auto X=1
run C10 t256g16k64 TTC_GREEDY_T=256 TTC_GREEDY_G=16 TTC_RING_KB=64
run C200 auto X=1
run C200 sm96 TTC_RING_SM_KB=96
done
cat $out
