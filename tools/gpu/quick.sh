# quick check: full GPU tests, c1/c3/c2 bench lines (device legs only)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log
B="--no-cpu-baseline --no-e2e"
timeout 300 python bench.py $B --steps 5 > gpurun_out/q_c1.json 2> gpurun_out/q_c1.err
timeout 300 python bench.py $B --config c3 --steps 2 --warmup 3 --iters 20 > gpurun_out/q_c3.json 2> gpurun_out/q_c3.err
timeout 600 python bench.py $B --config c2 --steps 3 --warmup 3 > gpurun_out/q_c2.json 2> gpurun_out/q_c2.err
echo done
