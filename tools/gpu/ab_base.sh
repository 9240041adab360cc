# session-4 baseline: GPU tests + bench lines at HEAD (split and per-bin schedules)
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s4_pytest.log
timeout 600 python bench.py > gpurun_out/s4_c1.json 2> gpurun_out/s4_c1.err; echo "rc=$?" >> gpurun_out/s4_c1.err
for c in c1 c2 c3; do
FM_SCHEDULE=bin timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/s4_bin_$c.json 2> gpurun_out/s4_bin_$c.err
done
for c in c2 c3; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/s4_$c.json 2> gpurun_out/s4_$c.err
done
echo done
