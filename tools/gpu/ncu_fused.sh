# ncu --set full of the first k_bpass / k_hpass / k_gpass launches of a config ($1, default c1)
c=${1:-c1}
ncu --set full --clock-control none --import-source on -k regex:"k_hpass|k_gpass|k_bpass" -c 3 \
  -o gpurun_out/ncu_fused_$c -f python bench.py --config $c --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fused_$c.log 2>&1
echo done
