timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2h.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2h.log
for c in c1 c2 c3; do
  it=""; [ "$c" = "c3" ] && it="--iters 20"
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 $it --no-cpu-baseline --no-e2e > gpurun_out/r2h_$c.json 2> gpurun_out/r2h_$c.err
done
ncu --set full --clock-control none --import-source on -k regex:"k_hpass|k_gpass|k_bpass" -c 3 -o gpurun_out/ncu_fused3_c2 -f python bench.py --config c2 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fused3_c2.log 2>&1
echo done
