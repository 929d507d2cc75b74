# ncu --set full of one k_sweeps launch (source-level, -lineinfo) for a workload: tools/gpu_ncu_src.sh <tag> <workload>
mkdir -p gpurun_out; tag=$1; wl=${2:-D20}
timeout 300 python tools/one_solve.py $wl 1 > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweeps -c 1 -o gpurun_out/${tag} python tools/one_solve.py $wl 1 > gpurun_out/${tag}_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/${tag}_ncu.log
