# after k_lambda_tc: the driver's round-end sequence, then the c3 lines and an ncu capture of k_lambda_tc
bash tools/gpu/roundend.sh
mkdir -p gpurun_out/r2f
O=gpurun_out/r2f
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c3 --shard --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_shard.json 2> $O/bench_c3_shard.err
A3="--config c3 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file $O/launches_c3.csv python bench.py $A3 > $O/ncu_a3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lambda_tc" -s 6 -c 1 -o $O/prof_c3_lam python bench.py $A3 > $O/ncu_l.log 2>&1
if [ -f $O/prof_c3_lam.ncu-rep ]; then
  python tools/ncu_summary.py $O/prof_c3_lam.ncu-rep > $O/prof_c3_lam.summary.md 2>&1
  rm -f $O/prof_c3_lam.ncu-rep
fi
echo done
