ARGS="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/launches_c1_v2.csv python bench.py $ARGS > gpurun_out/ncu3a.log 2>&1 ; \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_front|k_hstats|k_back|k_wupdate" -s 12 -c 4 -o gpurun_out/prof_c1_v2 python bench.py $ARGS > gpurun_out/ncu3b.log 2>&1
ARGS2="--config c2 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS2 > gpurun_out/plain3c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_front" -s 3 -c 1 -o gpurun_out/prof_c2_front python bench.py $ARGS2 > gpurun_out/ncu3c.log 2>&1
echo done
