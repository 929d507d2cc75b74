# A/B/n of library variants on bench workloads: each variant "label|ENV=..|lib" (lib relative to repo)
# usage: VARIANTS="a||paper_1903_11554_b200/libttcross.so b|TTC_NO_TMA=1|paper_1903_11554_b200/libttcross.so" \
#        WLS="D20 C200" tools/gpu_abn.sh <tag> [pytest -k expr]
mkdir -p gpurun_out; tag=$1; kexpr=$2
if [ -n "$kexpr" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
  tail -3 gpurun_out/${tag}_pytest.log
fi
for rep in 1 2; do for w in ${WLS:-D20 C200}; do for v in $VARIANTS; do
  IFS='|' read -r label envs lib <<< "$v"
  out=$(env $(echo "$envs" | tr "," " ") TTC_LIB_PATH=$PWD/$lib timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), d["integral"]["value"], round(d["roofline"].get("frac") or 0,4), d["launch_shape"])' 2>&1)
  echo "$rep $w $label $out"
done; done; done > gpurun_out/${tag}_ab.log 2>&1
cat gpurun_out/${tag}_ab.log
