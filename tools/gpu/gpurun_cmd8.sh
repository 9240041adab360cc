ARGS="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain8.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gain|k_vacc|k_ip|k_back|k_wstats|k_hstats" -s 25 -c 8 -o gpurun_out/prof_c1_v5 python bench.py $ARGS > gpurun_out/ncu8.log 2>&1
echo done
