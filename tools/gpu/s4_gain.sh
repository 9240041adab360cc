# k_gain_w (register accumulation) vs k_gain at c3; parity
timeout 600 python -m pytest tests/test_gpu_vtc.py tests/test_gpu_fullshape.py -x -q > gpurun_out/s4_gain_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s4_gain_pytest.log
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_gain_w.json 2> gpurun_out/s4_gain_w.err
FM_GAIN=cta timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_gain_cta.json 2> gpurun_out/s4_gain_cta.err
for g in 3 8; do
FM_GSEG=$g timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_gain_w_g$g.json 2> gpurun_out/s4_gain_w_g$g.err
done
echo done
