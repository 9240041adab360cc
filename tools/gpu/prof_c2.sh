A2="--config c2 --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py $A2 > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_phi|k_gain|k_ip" -s 6 -c 3 -o gpurun_out/prof_c2 python bench.py $A2 > gpurun_out/ncu_c2.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_c2.ncu-rep > gpurun_out/prof_c2.summary.md 2>&1
for k in k_phi k_gain k_ip; do python tools/ncu_lines.py gpurun_out/prof_c2.ncu-rep "$k" 10 >> gpurun_out/prof_c2.lines.txt 2>/dev/null; done
ncu -i gpurun_out/prof_c2.ncu-rep --page raw --csv > gpurun_out/prof_c2.raw.csv 2>/dev/null
rm -f gpurun_out/prof_c2.ncu-rep
echo done
