# final check of a freshly built library without the ncu passes: tools/gpu_evidence_quick.sh <tag>
mkdir -p gpurun_out; tag=$1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 600 python bench.py > gpurun_out/${tag}_bench_d20.jsonl 2> gpurun_out/${tag}_bench_d20.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --workload C200 --no-cpu-baseline > gpurun_out/${tag}_bench_c200.jsonl 2>&1
timeout 600 python bench.py --workload D5 --no-cpu-baseline > gpurun_out/${tag}_bench_d5.jsonl 2>&1
tail -2 gpurun_out/${tag}_smoke.log; tail -2 gpurun_out/${tag}_pytest.log; head -c 300 gpurun_out/${tag}_bench_d20.jsonl; echo; head -c 300 gpurun_out/${tag}_bench_c200.jsonl; echo; head -c 300 gpurun_out/${tag}_bench_d5.jsonl
