timeout 900 python -m pytest tests/test_gpu_fullrank.py -x -q > gpurun_out/pytest_fr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fr.log
echo done
