timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2n.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2n.log
timeout 600 python tools/parity_report.py gpurun_out/parity_r2n.json > gpurun_out/parity_r2n.log 2>&1
for c in c1 c4; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2n_$c.json 2> gpurun_out/r2n_$c.err
done
timeout 600 ncu --set full --clock-control none -k regex:"k_wiener_t|k_qinv" -c 2 -o gpurun_out/prof_wt -f python tools/dbg/wiener_c1.py > gpurun_out/ncu_wt.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_wt.ncu-rep > gpurun_out/prof_wt.summary.md 2>&1; rm -f gpurun_out/prof_wt.ncu-rep
echo done
