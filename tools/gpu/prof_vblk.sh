# ncu --set full of k_vacc_blk at c1 (M=8) and c3 (M=16), each after a clean run
A1="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
A3="--config c3 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $A1 > gpurun_out/plain_v1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc_blk" -s 12 -c 1 -o gpurun_out/prof_c1_vblk python bench.py $A1 > gpurun_out/ncu_v1.log 2>&1
timeout 300 python bench.py $A3 > gpurun_out/plain_v3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc_blk" -s 2 -c 1 -o gpurun_out/prof_c3_vblk python bench.py $A3 > gpurun_out/ncu_v3.log 2>&1
echo done
