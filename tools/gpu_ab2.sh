# correctness of the product build on the key cases, then A/B bench of product vs build/libttcross_head.so
mkdir -p gpurun_out; tag=${1:-ab}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "${2:-baseline_configs_full or small or D20 or streamed}" > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
WLS=${WLS:-"D20 C200 C10 D5"}
for rep in 1 2; do for w in $WLS; do
  for lib in paper_1903_11554_b200/libttcross.so build/libttcross_head.so; do
    echo "$rep $w $lib $(TTC_LIB_PATH=$PWD/$lib timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), d["integral"]["value"])')"
  done
done; done > gpurun_out/${tag}_ab.log 2>&1
timeout 300 python tools/probe_phases.py D20 --log > gpurun_out/${tag}_phases.jsonl 2>&1
tail -2 gpurun_out/${tag}_pytest.log; cat gpurun_out/${tag}_ab.log
