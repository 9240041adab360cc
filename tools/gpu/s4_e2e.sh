# e2e breakdown and host profile of the public run() call at config 1
timeout 300 python tools/e2e_breakdown.py --bench-like > gpurun_out/s4_e2e_breakdown.txt 2>&1
BENCH_E2E_PROFILE=1 timeout 600 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/s4_e2e_prof.json 2> gpurun_out/s4_e2e_prof.err
echo done
