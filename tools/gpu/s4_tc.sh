# tensor-core V at c3: which side bounds it (FM_VTC_DBG 1 = no MMAs, 2 = no operand build), c0 schedules
for dbg in 0 1 2; do
FM_VACC=tc FM_VTC_DBG=$dbg timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_tc_dbg$dbg.json 2> gpurun_out/s4_tc_dbg$dbg.err
done
FM_SCHEDULE=bin timeout 600 python bench.py --config c0 --no-cpu-baseline --no-e2e > gpurun_out/s4_bin_c0.json 2> gpurun_out/s4_bin_c0.err
timeout 600 python bench.py --config c0 --no-cpu-baseline --no-e2e > gpurun_out/s4_c0.json 2> gpurun_out/s4_c0.err
echo done
