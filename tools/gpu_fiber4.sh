# r02l: k_fiber_wsum (last-block reduction, grouped entries) ncu --set full on D_20 and C_200
mkdir -p gpurun_out
for w in D20 C200; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fiber_wsum -c 1 -o /tmp/fw_$w -f \
  python tools/one_solve.py $w 1 > gpurun_out/r02l_ncu_$w.log 2>&1
python tools/ncu_report.py /tmp/fw_$w.ncu-rep "r02l: k_fiber_wsum, $w quadrature (last-block reduction, grouped entries), ncu --set full --clock-control none" > gpurun_out/r02l_ncu_fiber_wsum_$w.txt 2>&1
done
grep -h "Duration\|pipe_fp64\|Issue Slots\|barrier:\|wait:\|Achieved Occ" gpurun_out/r02l_ncu_fiber_wsum_*.txt
