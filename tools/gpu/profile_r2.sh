# Round-2 artifacts: parity report, bench lines (every config, both schedules, sharded c3),
# reference-arm lines (unmodified fastsep), the c1 launch list, ncu --set full summaries.
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 600 python tools/parity_report.py $O/parity.json > $O/parity.log 2>&1
timeout 900 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
for c in c2 c4 c4mh c0; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c3 --shard --steps 2 --warmup 3 --iters 20 --no-e2e --no-cpu-baseline > $O/bench_c3_shard.json 2> $O/bench_c3_shard.err
for c in c1 c2 c3; do
  it=""; [ "$c" = "c3" ] && it="--iters 20"
  FM_SCHEDULE=fused timeout 600 python bench.py --config $c --steps 3 --warmup 3 $it --no-e2e --no-cpu-baseline > $O/bench_fused_$c.json 2> $O/bench_fused_$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_c1.json 2> $O/ref_c1.err
timeout 900 python bench.py --impl reference --config c2 --steps 3 --warmup 3 > $O/ref_c2.json 2> $O/ref_c2.err
timeout 900 python bench.py --impl reference --config c4mh --steps 2 --warmup 2 > $O/ref_c4mh.json 2> $O/ref_c4mh.err
timeout 900 python bench.py --impl reference --config c0 --steps 5 --warmup 3 > $O/ref_c0.json 2> $O/ref_c0.err
timeout 1200 python bench.py --impl reference --config c3 --steps 1 --warmup 1 > $O/ref_c3.json 2> $O/ref_c3.err
ARGS="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 80 --csv --log-file $O/launches_c1.csv python bench.py $ARGS > $O/ncu_a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc|k_back|k_ip" -s 12 -c 3 -o $O/prof_c1 python bench.py $ARGS > $O/ncu_b.log 2>&1
A3="--config c3 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_vacc_blk|k_back|k_wstats|k_hstats|k_gain|k_phi|k_ip" -s 20 -c 7 -o $O/prof_c3 python bench.py $A3 > $O/ncu_c.log 2>&1
A4="--config c4 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dp_latent" -s 4 -c 1 -o $O/prof_c4 python bench.py $A4 > $O/ncu_d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_wiener" -c 1 -o $O/prof_wiener python tools/dbg/wiener_c1.py > $O/ncu_e.log 2>&1
A2="--config c2 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_back|k_gain|k_vacc|k_ip" -s 12 -c 4 -o $O/prof_c2 python bench.py $A2 > $O/ncu_f.log 2>&1
FM_SCHEDULE=fused timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hpass|k_gpass|k_bpass" -s 3 -c 3 -o $O/prof_c2_fused python bench.py $A2 > $O/ncu_g.log 2>&1
for r in prof_c1 prof_c3 prof_c4 prof_wiener prof_c2 prof_c2_fused; do
  if [ -f $O/$r.ncu-rep ]; then
    python tools/ncu_summary.py $O/$r.ncu-rep > $O/$r.summary.md 2>&1
    ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
    ncu -i $O/$r.ncu-rep --page details --csv > $O/$r.details.csv 2>/dev/null
    rm -f $O/$r.ncu-rep
  fi
done
du -sh gpurun_out
echo done
