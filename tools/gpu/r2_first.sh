# round 2 first check: full GPU tests (incl. the new full-shape and drop-in tests), c1 bench
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_r2a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2a.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/r2a_c1.json 2> gpurun_out/r2a_c1.err
echo done
