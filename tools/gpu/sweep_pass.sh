# FM_PASS_CTAS / FM_PASS_S sweep of the fused passes (kernel ms from bench.py)
for c in c1 c3 c2; do
  for n in 444 1184 2368 4736; do
    for s in 0 2; do
      it="--iters 20"
      FM_PASS_CTAS=$n FM_PASS_S=$s timeout 300 python bench.py --config $c --steps 2 --warmup 3 $it --no-cpu-baseline --no-e2e > gpurun_out/sw_${c}_${n}_$s.json 2>/dev/null
      python tools/show.py gpurun_out/sw_${c}_${n}_$s.json >> gpurun_out/sweep.txt 2>&1
    done
  done
done
echo done
