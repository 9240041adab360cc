ARGS="--config c3 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain18.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc_tc" -s 2 -c 1 -o gpurun_out/prof_vtc16 python bench.py $ARGS > gpurun_out/ncu18.log 2>&1
echo done
