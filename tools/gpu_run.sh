#!/bin/bash
# one gpurun call: GPU tests (optionally filtered), fp64 peak probe, default bench
# usage: tools/gpu_run.sh <tag> [pytest -k expr]
tag=$1; kexpr=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [ -n "$kexpr" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
else
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
fi
[ -x tools/fp64_peak ] && timeout 120 tools/fp64_peak > gpurun_out/${tag}_fp64_peak.jsonl 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
tail -3 gpurun_out/${tag}_pytest.log; cat gpurun_out/${tag}_bench.jsonl | head -c 3000
