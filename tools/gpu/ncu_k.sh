# ncu --set full of the first launches matching $2 in config $1: tools/gpu/ncu_k.sh c1 "k_bpass|k_hpass" [count]
c=${1:-c1}; k=${2:-k_bpass}; n=${3:-2}
ncu --set full --clock-control none --import-source on -k regex:"$k" -c $n \
  -o gpurun_out/ncu_${c}_$(echo $k | tr -c 'a-z0-9\n' '_') -f python bench.py --config $c --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${c}.log 2>&1
echo done
