# tensor-core V at c3: skeleton only (3), no build + one MMA of three (6)
for dbg in 3 6; do
FM_VACC=tc FM_VTC_DBG=$dbg timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/s4_tc_dbg$dbg.json 2> gpurun_out/s4_tc_dbg$dbg.err
done
echo done
