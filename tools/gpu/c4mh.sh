timeout 900 python -m pytest tests/test_gpu_dp_mh.py tests/test_gpu_dp.py -x -q > gpurun_out/pytest_mh.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mh.log
B="--no-cpu-baseline --no-e2e"
timeout 600 python bench.py $B --config c4mh --steps 3 --warmup 3 > gpurun_out/c4mh.json 2> gpurun_out/c4mh.err
timeout 600 python bench.py $B --config c4 --steps 3 --warmup 3 > gpurun_out/c4.json 2> gpurun_out/c4.err
ARGS="--config c4 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py $ARGS > gpurun_out/ncu_c4.log 2>&1
echo done
