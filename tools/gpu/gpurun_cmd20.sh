# correctness of the tensor-core V at M = 16 against the oracle (per-op + a short c3-shaped run)
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
FM_VACC=simt timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_simt.json 2> gpurun_out/bench_c3.err
echo done
