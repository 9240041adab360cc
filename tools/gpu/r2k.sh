timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2k.log
for c in c1 c2; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_$c.json 2> gpurun_out/r2k_$c.err
done
echo done
