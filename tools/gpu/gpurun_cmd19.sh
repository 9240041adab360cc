for D in 0 1 2; do
FM_VTC_DBG=$D timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_c1_d$D.json 2> gpurun_out/bench_c1.err
FM_VTC_DBG=$D timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_d$D.json 2> gpurun_out/bench_c3.err
done
echo done
