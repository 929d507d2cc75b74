# round-2 evidence in one gpurun call (tag r02i): smoke, full GPU tests, default bench (D_20,
# with the all-core oracle cpu_baseline), the other t-form configs, the reference arm, the
# launch list of the default bench, one ncu --set full capture each of k_sweeps and
# k_fiber_wsum on D_20 (summaries + traffic written to gpurun_out), the per-phase log.
mkdir -p gpurun_out; tag=${1:-r02i}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_d20.jsonl 2> gpurun_out/${tag}_bench_d20.err
for w in C200 C10 D5 C4; do timeout 600 python bench.py --workload $w --no-cpu-baseline 2>/dev/null | tail -1; done > gpurun_out/${tag}_bench_other.jsonl
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_list.log 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_launches.csv "${tag}: D_20 bench (bench.py --steps 2 --warmup 3 --no-cpu-baseline), launch list (ncu, cold-cache, serialised)" > gpurun_out/${tag}_launches_d20.txt 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sweeps|k_fiber_wsum" -c 2 -o /tmp/${tag}_full \
  python tools/one_solve.py D20 1 > gpurun_out/${tag}_ncu_full.log 2>&1
python tools/ncu_report.py /tmp/${tag}_full.ncu-rep "${tag}: k_sweeps, one D_20 solve (64 Alg. 6 sweeps, persistent), ncu --set full --clock-control none" --kernel k_sweeps > gpurun_out/${tag}_ncu_k_sweeps_d20.txt 2>&1
python tools/ncu_report.py /tmp/${tag}_full.ncu-rep "${tag}: k_fiber_wsum, D_20 quadrature, ncu --set full --clock-control none" --kernel k_fiber_wsum > gpurun_out/${tag}_ncu_fiber_wsum_d20.txt 2>&1
python tools/probe_phases.py D20 --log > gpurun_out/${tag}_phases_d20.jsonl 2>&1
tail -2 gpurun_out/${tag}_pytest.log; tail -1 gpurun_out/${tag}_smoke.log; head -c 300 gpurun_out/${tag}_bench_d20.jsonl
