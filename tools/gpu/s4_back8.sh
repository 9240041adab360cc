# k_back_tc forced at M = 8 (config 1) against the SIMT k_back
FM_BACK=tc timeout 300 python -m pytest tests/test_gpu_run.py -x -q -k "c1 or c0_c64" > gpurun_out/s4_back8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s4_back8_pytest.log
FM_BACK=tc timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s4_c1_backtc.json 2> gpurun_out/s4_c1_backtc.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s4_c1_base.json 2> gpurun_out/s4_c1_base.err
echo done
