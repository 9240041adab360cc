timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2m.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2m.log
for c in c2 c0; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2m_$c.json 2> gpurun_out/r2m_$c.err
done
echo done
