# tensor-core projection k_back_tc: parity (every M > 8, full-shape c3), c3 timing vs FM_BACK=simt
timeout 900 python -m pytest tests/test_gpu_vtc.py tests/test_gpu_fullshape.py tests/test_gpu_bin.py -x -q > gpurun_out/s4_back_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s4_back_pytest.log
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/s4_c3_backtc.json 2> gpurun_out/s4_c3_backtc.err
FM_BACK=simt timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/s4_c3_backsimt.json 2> gpurun_out/s4_c3_backsimt.err
echo done
