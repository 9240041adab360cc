B="--no-cpu-baseline --no-e2e --steps 5"
for g in 1 2 3 4 6; do FM_GSEG=$g timeout 300 python bench.py $B > gpurun_out/seg_$g.json 2>> gpurun_out/seg.err; done
timeout 300 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > gpurun_out/seg_c3.json 2>> gpurun_out/seg.err
echo done
