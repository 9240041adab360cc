timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q -s > gpurun_out/pytest_pipe.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pipe.log
echo done
