ARGS="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_front|k_back|k_lambda|k_wstats|k_hstats|k_phi" -s 20 -c 7 -o gpurun_out/prof_c1_v3 python bench.py $ARGS > gpurun_out/ncu5.log 2>&1
echo done
