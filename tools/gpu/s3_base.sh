# session-3 baseline: GPU tests + default bench at HEAD
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s3_pytest.log
timeout 600 python bench.py > gpurun_out/s3_bench_c1.json 2> gpurun_out/s3_bench_c1.err; echo "rc=$?" >> gpurun_out/s3_bench_c1.err
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/s3_bench_c3.json 2> gpurun_out/s3_bench_c3.err
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/s3_bench_c2.json 2> gpurun_out/s3_bench_c2.err
echo done
