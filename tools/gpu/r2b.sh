# round 2: GPU tests after the fused-pass rewrite
timeout 1500 python -m pytest tests -m gpu -q --maxfail=15 --durations=10 > gpurun_out/pytest_r2b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2b.log
