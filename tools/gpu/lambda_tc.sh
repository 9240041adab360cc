# k_lambda_tc: parity (full-shape c3, K = 8 / 16 / 32 forced on small shapes) and c3 timing; sharded line
FM_LAMBDA=tc timeout 600 python -m pytest tests/test_gpu_vtc.py tests/test_gpu_run.py -x -q > gpurun_out/s4_lam_pytest_forced.log 2>&1; echo "rc=$?" >> gpurun_out/s4_lam_pytest_forced.log
timeout 600 python -m pytest tests/test_gpu_fullshape.py -x -q > gpurun_out/s4_lam_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s4_lam_pytest.log
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_lam_tc.json 2> gpurun_out/s4_lam_tc.err
FM_LAMBDA=simt timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_lam_simt.json 2> gpurun_out/s4_lam_simt.err
FM_LAMBDA=tc timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_lam_c1tc.json 2> gpurun_out/s4_lam_c1tc.err
timeout 300 python bench.py --config c3 --shard --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_lam_shard.json 2> gpurun_out/s4_lam_shard.err
echo done
