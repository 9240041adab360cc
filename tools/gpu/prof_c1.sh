# ncu --set full of one launch of each c1 kernel (after a clean run)
A1="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $A1 > gpurun_out/plain_c1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_ip|k_back|k_gain|k_wstats|k_hstats|k_phi|k_lambda|k_vacc" -s 40 -c 9 -o gpurun_out/prof_c1_all python bench.py $A1 > gpurun_out/ncu_c1_all.log 2>&1
echo done
