# A/B of two library builds (TTC_LIB_PATH) on the given t-form configs, interleaved, 2 rounds
mkdir -p gpurun_out
WLS=${WLS:-"D20 C200 C10 D5"}
for rep in 1 2; do for w in $WLS; do
  for lib in paper_1903_11554_b200/libttcross.so build/libttcross_head.so; do
    echo "$rep $w $lib $(TTC_LIB_PATH=$PWD/$lib python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
  done
done; done > gpurun_out/ab.log 2>&1
