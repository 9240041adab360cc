timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 300 python tools/phase_timing.py c1 > gpurun_out/phase_c1.txt 2>&1
timeout 300 python tools/phase_timing.py c3 > gpurun_out/phase_c3.txt 2>&1
echo done
