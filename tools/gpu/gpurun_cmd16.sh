# tensor-core V accumulation: quick parity first, then the whole suite and benches
timeout 300 python -m pytest tests/test_gpu_run.py -q -x --timeout 120 -k "config0_c64 or config1_c64" > gpurun_out/pytest_tc.log 2>&1; echo rc=$? >> gpurun_out/pytest_tc.log
if grep -q "rc=0" gpurun_out/pytest_tc.log; then
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
FM_VACC=simt timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_simt.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
fi
echo done
