# per-bin schedule: tests, then c2/c0 A/B against split
timeout 900 python -m pytest tests/test_gpu_bin.py tests/test_gpu_shard2.py tests/test_gpu_ipw.py -x -q > gpurun_out/s3_bin_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s3_bin_pytest.log
FM_SCHEDULE=bin timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/s3_bin_c2.json 2> gpurun_out/s3_bin_c2.err
FM_SCHEDULE=bin timeout 600 python bench.py --config c0 --no-cpu-baseline --no-e2e > gpurun_out/s3_bin_c0.json 2> gpurun_out/s3_bin_c0.err
timeout 600 python bench.py --config c0 --no-cpu-baseline --no-e2e > gpurun_out/s3_split_c0.json 2> gpurun_out/s3_split_c0.err
echo done
