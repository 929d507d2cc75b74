# cross-GPU wavefront loopback tests + the GPU suite + D_20 / C_200 bench: tools/gpu_peer.sh <tag>
mkdir -p gpurun_out; tag=$1
timeout 900 python -m pytest tests/test_gpu_peer.py -q -x > gpurun_out/${tag}_peer.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_peer.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/${tag}_bench_d20.jsonl 2>&1
timeout 600 python bench.py --workload C200 --steps 100 --no-cpu-baseline > gpurun_out/${tag}_bench_c200.jsonl 2>&1
tail -3 gpurun_out/${tag}_peer.log; tail -2 gpurun_out/${tag}_pytest.log; head -c 300 gpurun_out/${tag}_bench_d20.jsonl
