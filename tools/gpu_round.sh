# parity suite + bench lines of the t-form configs + per-phase probe (one gpurun call)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for w in D5 C10 D20 C200; do python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1; done > gpurun_out/bench_r.jsonl
python tools/probe_phases.py D5 D20 > gpurun_out/phases.jsonl 2>&1
