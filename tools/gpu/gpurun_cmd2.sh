timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config c0 --steps 5 --no-cpu-baseline > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err
echo done
