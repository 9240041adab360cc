# Round artifacts: parity report, bench lines (c1 default with every leg, reference arm, c3, c4),
# the c1 launch list and one ncu --set full capture of the c1 dominant kernel.
timeout 600 python tools/parity_report.py gpurun_out/parity.json > gpurun_out/parity.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c1_full.json 2> gpurun_out/bench_c1_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
ARGS="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain_pr.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 80 --csv --log-file gpurun_out/launches_c1.csv python bench.py $ARGS > gpurun_out/ncu_pr_a.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc|k_back|k_ip" -s 12 -c 3 -o gpurun_out/prof_c1 python bench.py $ARGS > gpurun_out/ncu_pr_b.log 2>&1
echo done
