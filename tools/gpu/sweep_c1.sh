# c1 knob sweep: V segments / V kernel / IP kernel
for v in "FM_GSEG=1" "FM_GSEG=2" "FM_GSEG=3" "FM_GSEG=4" "FM_VACC=blk" "FM_IP=w"; do
  env $v timeout 300 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s1.json 2>/dev/null
  echo "$v $(python tools/show.py gpurun_out/s1.json)" >> gpurun_out/sweep_c1.txt
done
echo done
