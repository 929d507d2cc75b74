mkdir -p gpurun_out
timeout 120 python tools/one_solve.py D20 2 > gpurun_out/r02d_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/r02d_plain.log
TTC_PHASE_JOB=9 timeout 120 python tools/one_solve.py D20 2 > gpurun_out/r02d_pj.log 2>&1; echo "pj rc=$?" >> gpurun_out/r02d_pj.log
timeout 600 /usr/local/cuda/bin/cuda-gdb -batch -ex "set cuda break_on_launch none" -ex run -ex "info cuda kernels" -ex "bt" -ex "info cuda lanes" -ex "x/8i \$pc-32" -ex "info line *\$pc" --args python tools/one_solve.py D20 1 > gpurun_out/r02d_gdb.log 2>&1
echo "gdb rc=$?" >> gpurun_out/r02d_gdb.log
tail -3 gpurun_out/r02d_plain.log gpurun_out/r02d_pj.log; tail -40 gpurun_out/r02d_gdb.log
