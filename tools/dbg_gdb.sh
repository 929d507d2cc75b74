# cuda-gdb batch run of one solve: tools/dbg_gdb.sh <tag> <workload> [ENV=..]
mkdir -p gpurun_out; tag=$1; wl=$2; shift 2
env "$@" timeout 600 /usr/local/cuda/bin/cuda-gdb -batch -ex "set cuda break_on_launch none" -ex run -ex "info cuda kernels" -ex "bt" -ex "x/12i \$pc-96" -ex "info line *\$pc" -ex "info registers" --args python tools/one_solve.py $wl 1 > gpurun_out/${tag}_gdb.log 2>&1
grep -n "Illegal\|exception\|Exception\|=>\|Line \|CUDA_EXCEPTION" gpurun_out/${tag}_gdb.log | head -20
