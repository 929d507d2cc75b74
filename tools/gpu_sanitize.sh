# compute-sanitizer evidence on the small paths: tools/gpu_sanitize.sh <tag>
# memcheck on smoke() (D_4, cached shape), on the small forced-TMA-ring parity cases and on two
# small parity cases; racecheck (shared-memory hazards) and synccheck on smoke().
mkdir -p gpurun_out; tag=$1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_plain_smoke.log 2>&1 || exit 1
timeout 500 $CS --tool memcheck --log-file gpurun_out/${tag}_memcheck_smoke.log python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_memcheck_smoke.out 2>&1; echo "rc=$?" >> gpurun_out/${tag}_memcheck_smoke.out
timeout 700 $CS --tool memcheck --log-file gpurun_out/${tag}_memcheck_ring.log python -m pytest tests/test_gpu_fullsize.py -q -k streamed_rook_steps_small > gpurun_out/${tag}_memcheck_ring.out 2>&1; echo "rc=$?" >> gpurun_out/${tag}_memcheck_ring.out
timeout 500 $CS --tool racecheck --log-file gpurun_out/${tag}_racecheck_smoke.log python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_racecheck_smoke.out 2>&1; echo "rc=$?" >> gpurun_out/${tag}_racecheck_smoke.out
timeout 500 $CS --tool synccheck --log-file gpurun_out/${tag}_synccheck_smoke.log python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_synccheck_smoke.out 2>&1; echo "rc=$?" >> gpurun_out/${tag}_synccheck_smoke.out
for f in gpurun_out/${tag}_*.out; do echo "== $f"; tail -3 $f; done
for f in gpurun_out/${tag}_*check*.log; do echo "== $f"; tail -4 $f; done
