# Re-verify after a container restore: GPU tests, smoke, c1 and c3 bench lines.
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo done
