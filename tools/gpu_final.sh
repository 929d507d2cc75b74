# round-end evidence in one gpurun call: parity suite, smoke, bench lines of every config
# (default D5 line with the oracle cpu_baseline), the reference arm, the D5 launch list and
# ncu --set full captures of k_sweeps (D5, D20) and k_fiber_wsum (D20)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f_pytest.log 2>&1
python bench.py > gpurun_out/f_bench_d5.jsonl 2> gpurun_out/f_bench_d5.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.jsonl 2>&1
for w in C4 C10 D20 C200 Dx8 Dx8f Cx64 Ex6; do
  python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
done > gpurun_out/f_bench_all.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_d5.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweeps -c 1 -o gpurun_out/f_sweeps_d5 -f \
  python bench.py --workload D5 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/f_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweeps -c 1 -o gpurun_out/f_sweeps_d20 -f \
  python bench.py --workload D20 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/f_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fiber_wsum -c 1 -o gpurun_out/f_fiber_d20 -f \
  python bench.py --workload D20 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/f_ncu3.log 2>&1
tail -1 gpurun_out/f_pytest.log
# summaries on the box (the captures themselves are too large to bring back together)
python tools/ncu_summary.py gpurun_out/f_launches_d5.csv "r01n: D_5 bench (bench.py --steps 5 --warmup 3 --no-cpu-baseline), launch list" > gpurun_out/f_launches_d5.txt
python tools/ncu_report.py gpurun_out/f_sweeps_d5.ncu-rep "r01n: k_sweeps, one D_5 solve (16 Alg. 6 sweeps, persistent), ncu --set full --clock-control none" > gpurun_out/f_ncu_k_sweeps_d5.txt 2>&1
python tools/ncu_report.py gpurun_out/f_sweeps_d20.ncu-rep "r01n: k_sweeps, one D_20 solve (64 Alg. 6 sweeps, persistent), ncu --set full --clock-control none" > gpurun_out/f_ncu_k_sweeps_d20.txt 2>&1
python tools/ncu_report.py gpurun_out/f_fiber_d20.ncu-rep "r01n: k_fiber_wsum, D_20 quadrature (tiled, cluster node split), ncu --set full --clock-control none" > gpurun_out/f_ncu_fiber_d20.txt 2>&1
ncu -i gpurun_out/f_sweeps_d5.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/f_d5_dram.csv 2>&1
ncu -i gpurun_out/f_sweeps_d20.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/f_d20_dram.csv 2>&1
rm -f gpurun_out/f_sweeps_d20.ncu-rep gpurun_out/f_fiber_d20.ncu-rep
