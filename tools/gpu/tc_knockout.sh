# new warp-specialised tensor-core V: parity, then c3 timing with the knock-outs
timeout 600 python -m pytest tests/test_gpu_vtc.py -x -q > gpurun_out/s4_tc3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s4_tc3_pytest.log
for dbg in 0 1 2 3; do
FM_VACC=tc FM_VTC_DBG=$dbg timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_tc3_dbg$dbg.json 2> gpurun_out/s4_tc3_dbg$dbg.err
done
echo done
