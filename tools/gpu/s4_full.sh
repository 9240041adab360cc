# full GPU suite with the new defaults (tensor-core V at even M >= 10, per-bin schedule for large batches),
# c2 schedule crossover by batch size, c3 / c2 bench lines
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s4_full_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s4_full_pytest.log
for b in 8 16 32 64; do
for sch in split bin; do
FM_SCHEDULE=$sch timeout 300 python bench.py --config c2 --mixtures $b --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/s4_c2_${sch}_b$b.json 2> gpurun_out/s4_c2_${sch}_b$b.err
done; done
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/s4_c3_tc.json 2> gpurun_out/s4_c3_tc.err
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/s4_c2_def.json 2> gpurun_out/s4_c2_def.err
echo done
