timeout 600 python -m pytest tests/test_gpu_vtc.py -x -q > gpurun_out/pytest_q1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q1.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/q1_c1.json 2> gpurun_out/q1_c1.err
FM_VACC=simt timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/q1_c1s.json 2>> gpurun_out/q1_c1.err
echo done
