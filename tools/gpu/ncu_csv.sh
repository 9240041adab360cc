# ncu --set full of launches matching $1 at c1 (skip $2, count $3); raw / SASS pages come back as CSV
k=${1:-k_vacc}; s=${2:-4}; n=${3:-1}; tag=${4:-k}
A1="--steps 1 --warmup 3 --iters 5 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c $n -f -o /tmp/prof_$tag python bench.py $A1 > gpurun_out/ncu_$tag.log 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_sass.csv 2>/dev/null
echo done
