# round evidence: full GPU tests, default bench (D_20) + C_200 + D_5, launch list and one
# ncu --set full capture of k_sweeps (D_20) and of the fiber kernel, smoke(): tools/gpu_evidence.sh <tag>
mkdir -p gpurun_out; tag=$1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench_d20.jsonl 2> gpurun_out/${tag}_bench_d20.err
timeout 600 python bench.py --workload C200 --no-cpu-baseline > gpurun_out/${tag}_bench_c200.jsonl 2>&1
timeout 600 python bench.py --workload D5 --no-cpu-baseline > gpurun_out/${tag}_bench_d5.jsonl 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.jsonl 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_list.log 2>&1
timeout 300 python tools/one_solve.py D20 1 > gpurun_out/${tag}_one.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sweeps|k_fiber_wsum" -c 2 -o gpurun_out/${tag}_full python tools/one_solve.py D20 1 > gpurun_out/${tag}_ncu_full.log 2>&1
tail -2 gpurun_out/${tag}_pytest.log; head -c 400 gpurun_out/${tag}_bench_d20.jsonl
