# c1: bench line, then ncu --set full of the V kernel (default and blocked); the
# reports stay on the box, their raw / SASS pages come back as CSV
B="--no-cpu-baseline --no-e2e"
rm -f gpurun_out/c1.txt
for v in "FM_VACC=simt" "FM_VACC=blk"; do
  env $v timeout 300 python bench.py $B --steps 5 > gpurun_out/c1_ab.json 2> gpurun_out/c1_ab.err
  echo "$v $(python tools/show.py gpurun_out/c1_ab.json)" >> gpurun_out/c1.txt
done
A1="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
FM_VACC=simt timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vacc|k_gain" -s 8 -c 2 -f -o /tmp/prof_c1_vacc python bench.py $A1 > gpurun_out/ncu_c1_vacc.log 2>&1
FM_VACC=blk timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vacc" -s 4 -c 1 -f -o /tmp/prof_c1_blk python bench.py $A1 > gpurun_out/ncu_c1_blk.log 2>&1
for r in prof_c1_vacc prof_c1_blk; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_sass.csv 2>/dev/null
done
echo done
