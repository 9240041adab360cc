ARGS="--config c4mh --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dp_mh" -s 4 -c 1 -o gpurun_out/prof_mh python bench.py $ARGS > gpurun_out/ncu_mh.log 2>&1
echo done
