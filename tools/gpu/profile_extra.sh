# ncu --set full of the c3 tensor-core V kernel and the c4 latent kernel (each after a clean run)
A3="--config c3 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
A4="--config c4 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $A3 > gpurun_out/plain_x3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc_tc" -s 2 -c 1 -o gpurun_out/prof_c3_vtc python bench.py $A3 > gpurun_out/ncu_x3.log 2>&1
timeout 300 python bench.py $A4 > gpurun_out/plain_x4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dp_latent" -s 1 -c 1 -o gpurun_out/prof_c4_latent python bench.py $A4 > gpurun_out/ncu_x4.log 2>&1
timeout 300 python bench.py $A4 > gpurun_out/plain_x4b.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 100 --csv --log-file gpurun_out/launches_c4.csv python bench.py $A4 > gpurun_out/ncu_x4b.log 2>&1
echo done
