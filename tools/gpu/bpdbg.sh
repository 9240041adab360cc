# k_bpass component timing: FM_BP_DBG bit 0 skip W statistics, 1 lambda tile, 2 projection, 3 phi
for c in c1 c3 c2; do
  for d in 0 1 2 4 8 15; do
    FM_BP_DBG=$d timeout 300 python bench.py --config $c --steps 2 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e > gpurun_out/bd_${c}_$d.json 2>/dev/null
    echo "$c dbg=$d $(python -c "import json;d=json.load(open('gpurun_out/bd_${c}_$d.json'));print(round(d['roofline']['kernel_ms']['k_bpass']*1e3,1))" 2>&1)" >> gpurun_out/bpdbg.txt
  done
done
echo done
