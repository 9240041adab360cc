timeout 600 python tools/parity_report.py gpurun_out/parity.json > gpurun_out/parity.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c1_full.json 2> gpurun_out/bench_c1_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ARGS="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain9.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 80 --csv --log-file gpurun_out/launches_c1.csv python bench.py $ARGS > gpurun_out/ncu9a.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc|k_back|k_gain" -s 12 -c 3 -o gpurun_out/prof_c1_r1 python bench.py $ARGS > gpurun_out/ncu9b.log 2>&1
echo done
