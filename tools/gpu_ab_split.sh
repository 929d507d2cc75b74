# A/B of the split-start persistent loop (TTC_SPLIT_WAIT=1, product build) against the same
# source with -DTTC_SPLIT_WAIT=0 (build/libttcross_nosplit.so), interleaved; then the parity
# tests that cover the persistent loop (build/libttcross_head.so, when present: the previous commit's build)
mkdir -p gpurun_out; tag=${1:-split}
WLS=${WLS:-"D20 C200 C10 D5"}
for rep in 1 2; do for w in $WLS; do
  for lib in paper_1903_11554_b200/libttcross.so build/libttcross_nosplit.so build/libttcross_head.so; do
    echo "$rep $w $lib $(TTC_LIB_PATH=$PWD/$lib timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["integral"]["value"])')"
  done
done; done > gpurun_out/${tag}_ab.log 2>&1
cat gpurun_out/${tag}_ab.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
tail -5 gpurun_out/${tag}_pytest.log
