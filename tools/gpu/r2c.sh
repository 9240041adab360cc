# round 2: bench lines of every config after the fused-pass rewrite + reference arm c1
for c in c1 c2 c3 c4 c4mh; do
  it=""; [ "$c" = "c3" ] && it="--iters 20"
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 $it --no-cpu-baseline > gpurun_out/r2c_$c.json 2> gpurun_out/r2c_$c.err
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2c_ref_c1.json 2> gpurun_out/r2c_ref_c1.err
echo done
