mkdir -p gpurun_out
timeout 120 python tools/one_solve.py D20 2 > gpurun_out/r02e_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/r02e_plain.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "D20 or streamed" > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02e_pytest.log
timeout 300 python tools/probe_phases.py D20 C200 --log > gpurun_out/r02e_phases.jsonl 2>&1
TTC_PHASE_JOB=1 timeout 300 python tools/probe_phases.py D20 --log > gpurun_out/r02e_phases_j1.jsonl 2>&1
tail -3 gpurun_out/r02e_plain.log gpurun_out/r02e_pytest.log
