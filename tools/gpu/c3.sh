timeout 600 python -m pytest tests/test_gpu_vtc.py tests/test_gpu_ops.py -x -q > gpurun_out/pytest_c3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c3.log
timeout 300 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > gpurun_out/c3x.json 2> gpurun_out/c3x.err
echo done
