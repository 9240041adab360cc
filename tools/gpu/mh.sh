timeout 900 python -m pytest tests/test_gpu_dp_mh.py tests/test_gpu_dp.py -x -q > gpurun_out/pytest_mh.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mh.log
echo done
