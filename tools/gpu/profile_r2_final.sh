# Final round-2 artefacts: parity report, bench lines (every config; A/B lines for the kernels that
# changed defaults), reference arm (c1, c0), launch lists, ncu --set full summaries.
mkdir -p gpurun_out/r2f
O=gpurun_out/r2f
timeout 600 python tools/parity_report.py $O/parity.json > $O/parity.log 2>&1
timeout 900 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
for c in c0 c2 c3 c4 c4mh; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config c3 --shard --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_shard.json 2> $O/bench_c3_shard.err
FM_SCHEDULE=split timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_split.json 2> $O/bench_c2_split.err
FM_VACC=blk FM_BACK=simt timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_simt.json 2> $O/bench_c3_simt.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_c1.json 2> $O/ref_c1.err
timeout 900 python bench.py --impl reference --config c0 --steps 5 --warmup 3 > $O/ref_c0.json 2> $O/ref_c0.err
ARGS="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 80 --csv --log-file $O/launches_c1.csv python bench.py $ARGS > $O/ncu_a.log 2>&1
A3="--config c3 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file $O/launches_c3.csv python bench.py $A3 > $O/ncu_a3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc|k_back|k_ip" -s 12 -c 3 -o $O/prof_c1 python bench.py $ARGS > $O/ncu_b.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_vacc_tc|k_back_tc|k_wstats|k_hstats|k_gain|k_phi|k_ip|k_lambda" -s 27 -c 9 -o $O/prof_c3 python bench.py $A3 > $O/ncu_c.log 2>&1
A2="--config c2 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_binw|k_hstats" -s 6 -c 2 -o $O/prof_c2 python bench.py $A2 > $O/ncu_f.log 2>&1
for r in prof_c1 prof_c3 prof_c2; do
  if [ -f $O/$r.ncu-rep ]; then
    python tools/ncu_summary.py $O/$r.ncu-rep > $O/$r.summary.md 2>&1
    ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
    rm -f $O/$r.ncu-rep
  fi
done
du -sh gpurun_out
echo done
