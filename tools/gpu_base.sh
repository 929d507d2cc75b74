# check of a build: GPU tests, bench lines (D_20 default, C_200, C_10, D_5), per-phase probe of D_20
mkdir -p gpurun_out; tag=${1:-base}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench_d20.jsonl 2> gpurun_out/${tag}_bench_d20.err
for w in C200 C10 D5; do timeout 600 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1; done > gpurun_out/${tag}_bench_other.jsonl
timeout 600 python tools/probe_phases.py D20 --log > gpurun_out/${tag}_phases.jsonl 2>&1
tail -2 gpurun_out/${tag}_pytest.log; for f in gpurun_out/${tag}_bench_d20.jsonl gpurun_out/${tag}_bench_other.jsonl; do cut -c1-260 $f; done; head -1 gpurun_out/${tag}_phases.jsonl | cut -c1-600
