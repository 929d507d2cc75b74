mkdir -p gpurun_out
python tools/trace_steps.py D5 C10 > gpurun_out/trace.jsonl 2>&1
for w in D20 C200 D5; do python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1; done > gpurun_out/b3.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
