timeout 600 python -m pytest tests/test_gpu_stft.py -x -q > gpurun_out/pytest_stft.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stft.log
echo done
