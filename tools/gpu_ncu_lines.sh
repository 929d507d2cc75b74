# ncu --set full (source counters) of one k_sweeps launch + per-line stall summary on the box:
# tools/gpu_ncu_lines.sh <tag> <workload> <kernel mangled name>
mkdir -p gpurun_out; tag=$1; wl=${2:-D20}; kn=${3:-_ZN3ttc8k_sweepsILi1ELb0ELi256EEEvNS_6DevCtxEii}
timeout 300 python tools/one_solve.py $wl 1 > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_sweeps -c 1 -o /tmp/${tag} python tools/one_solve.py $wl 1 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
python tools/ncu_lines.py /tmp/${tag}.ncu-rep paper_1903_11554_b200/libttcross.so $kn 100 --func "${4:-extend_side_reg}" > gpurun_out/${tag}_lines.txt 2>&1
python tools/ncu_report.py /tmp/${tag}.ncu-rep "${tag}: k_sweeps ${wl}" > gpurun_out/${tag}_report.txt 2>&1
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source=sass 2>/dev/null | head -3 > gpurun_out/${tag}_srchdr.csv
head -60 gpurun_out/${tag}_lines.txt | cut -c1-250
