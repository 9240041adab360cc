timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2i.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2i.log
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2i_c1.json 2> gpurun_out/r2i_c1.err
echo done
