timeout 900 python -m pytest tests/test_gpu_dp_mh.py tests/test_gpu_dp.py tests/test_gpu_run.py -x -q > gpurun_out/pytest_dp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dp.log
B="--no-cpu-baseline --no-e2e --steps 3 --warmup 3"
timeout 600 python bench.py $B --config c4 > gpurun_out/dp_c4.json 2> gpurun_out/dp.err
timeout 600 python bench.py $B --config c4mh > gpurun_out/dp_c4mh.json 2>> gpurun_out/dp.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/dp_c1.json 2>> gpurun_out/dp.err
echo done
