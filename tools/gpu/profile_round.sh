# Round artifacts: parity report, bench lines (c1 default with every leg, reference arm, c2, c3,
# c4, c4mh), the c1 launch list, ncu --set full captures of the dominant kernels.
timeout 600 python tools/parity_report.py gpurun_out/parity.json > gpurun_out/parity.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c1_full.json 2> gpurun_out/bench_c1_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --iters 20 --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c4mh --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c4mh.json 2> gpurun_out/bench_c4mh.err
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python tools/e2e_breakdown.py --bench-like > gpurun_out/e2e_breakdown.txt 2>&1
ARGS="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain_pr.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 80 --csv --log-file gpurun_out/launches_c1.csv python bench.py $ARGS > gpurun_out/ncu_pr_a.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc|k_back|k_ip" -s 12 -c 3 -o gpurun_out/prof_c1 python bench.py $ARGS > gpurun_out/ncu_pr_b.log 2>&1
A3="--config c3 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $A3 > gpurun_out/plain_x3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vacc_blk" -s 2 -c 1 -o gpurun_out/prof_c3_vblk python bench.py $A3 > gpurun_out/ncu_x3.log 2>&1
A4="--config c4mh --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $A4 > gpurun_out/plain_x4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dp_mh" -s 4 -c 1 -o gpurun_out/prof_c4mh python bench.py $A4 > gpurun_out/ncu_x4.log 2>&1
# summarise the captures on the box (the .ncu-rep files exceed gpurun's copy-back limit)
for r in prof_c1 prof_c3_vblk prof_c4mh; do
  if [ -f gpurun_out/$r.ncu-rep ]; then
    python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.summary.md 2>&1
    for k in k_vacc k_back k_ip k_vacc_blk k_dp_mh; do
      python tools/ncu_lines.py gpurun_out/$r.ncu-rep "$k" 12 >> gpurun_out/$r.lines.txt 2>/dev/null
    done
    ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
    rm -f gpurun_out/$r.ncu-rep
  fi
done
du -sh gpurun_out
echo done
