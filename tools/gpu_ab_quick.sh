# quick interleaved A/B of library builds (TTC_LIB_PATH): tools/gpu_ab_quick.sh <tag> <lib>...
mkdir -p gpurun_out; tag=$1; shift
for rep in 1 2; do for w in ${WLS:-D20 C200}; do for lib in "$@"; do
  echo "$rep $w $lib $(TTC_LIB_PATH=$PWD/$lib timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["integral"]["value"])')"
done; done; done > gpurun_out/${tag}_ab.log 2>&1
cat gpurun_out/${tag}_ab.log
