# ncu --set full of the tensor-core kernels (c3) and the per-bin kernel (c2), summarised on the box
mkdir -p gpurun_out/s4
O=gpurun_out/s4
A3="--config c3 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_vacc_tc|k_back_tc|k_gain" -s 9 -c 3 -o $O/prof_c3_tc python bench.py $A3 > $O/ncu_c3.log 2>&1
A2="--config c2 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_binw|k_hstats" -s 6 -c 2 -o $O/prof_c2_bin python bench.py $A2 > $O/ncu_c2.log 2>&1
for r in prof_c3_tc prof_c2_bin; do
  if [ -f $O/$r.ncu-rep ]; then
    python tools/ncu_summary.py $O/$r.ncu-rep > $O/$r.summary.md 2>&1
    ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
    ncu -i $O/$r.ncu-rep --page source --csv > $O/$r.source.csv 2>/dev/null
    rm -f $O/$r.ncu-rep
  fi
done
du -sh gpurun_out
echo done
