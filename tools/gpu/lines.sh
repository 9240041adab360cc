# per-source-line stall profile of the kernels matching $1 at c1 (skip $2, count $3)
k=${1:-k_ip}; s=${2:-4}; n=${3:-1}; tag=${4:-k}
A1="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c $n -f -o /tmp/prof_$tag python bench.py $A1 > gpurun_out/ncu_$tag.log 2>&1
for kk in $(echo $k | tr '|' ' '); do
  python tools/ncu_lines.py /tmp/prof_$tag.ncu-rep $kk 40 > gpurun_out/lines_${tag}_$kk.txt 2>&1
done
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
echo done
