# launch-shape experiments after the ring-capacity shape search (r02c): auto vs forced shapes
mkdir -p gpurun_out
out=gpurun_out/shape3.log; : > $out
run() {  # workload label envs...
  w=$1; label=$2; shift 2
  r=$(env "$@" timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>gpurun_out/shape3_err_${w}_$label.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), d["integral"]["value"], round(d["roofline"].get("frac") or 0,4), d["launch_shape"])' 2>&1 | tail -1)
  echo "$w $label $r" >> $out
}
for rep in 1 2; do
run D20 auto X=1
run D20 t512g6k192 TTC_GREEDY_T=512 TTC_GREEDY_G=6 TTC_RING_KB=192
run D20 t512g5k192 TTC_GREEDY_T=512 TTC_GREEDY_G=5 TTC_RING_KB=192
run D20 t512g4k192 TTC_GREEDY_T=512 TTC_GREEDY_G=4 TTC_RING_KB=192
run D20 t256g8k96 TTC_GREEDY_T=256 TTC_GREEDY_G=8 TTC_RING_KB=96
run D20 t256g8k64 TTC_GREEDY_T=256 TTC_GREEDY_G=8 TTC_RING_KB=64
run D20 t512g6k128 TTC_GREEDY_T=512 TTC_GREEDY_G=6 TTC_RING_KB=128
run C200 auto X=1
run C200 t256g1k64 TTC_GREEDY_T=256 TTC_GREEDY_G=1 TTC_RING_KB=64
run C200 t256g1k96 TTC_GREEDY_T=256 TTC_GREEDY_G=1 TTC_RING_KB=96
done
run D5 auto X=1
run C10 auto X=1
cat $out
