timeout 600 python -m pytest tests/test_gpu_vtc.py -x -q > gpurun_out/pytest_q2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q2.log
B="--no-cpu-baseline --no-e2e"
FM_VACC=blk timeout 300 python bench.py $B --steps 5 > gpurun_out/q2_c1b.json 2> gpurun_out/q2.err
timeout 300 python bench.py $B --steps 5 > gpurun_out/q2_c1.json 2>> gpurun_out/q2.err
timeout 300 python bench.py $B --config c3 --steps 2 --warmup 3 --iters 20 > gpurun_out/q2_c3.json 2>> gpurun_out/q2.err
echo done
