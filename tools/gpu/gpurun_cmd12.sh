ARGS="--config c4 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain12.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dp_latent" -s 1 -c 1 -o gpurun_out/prof_c4_latent python bench.py $ARGS > gpurun_out/ncu12.log 2>&1
echo done
