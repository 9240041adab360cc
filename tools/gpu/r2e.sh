python tools/dbg/prologue.py > gpurun_out/dbg.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2e.log
for c in c1 c2 c3; do
  it=""; [ "$c" = "c3" ] && it="--iters 20"
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 $it --no-cpu-baseline --no-e2e > gpurun_out/r2e_$c.json 2> gpurun_out/r2e_$c.err
done
echo done
