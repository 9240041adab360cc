set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
ARGS="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches_c1.csv python bench.py $ARGS > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spatial -s 5 -c 1 -o gpurun_out/prof_spatial_c1 python bench.py $ARGS > gpurun_out/ncu2.log 2>&1
echo done
