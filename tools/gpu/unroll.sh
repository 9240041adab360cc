# graph unroll sweep at c1 (iterations captured per CUDA graph), device leg only
B="--no-cpu-baseline --no-e2e"
for u in 1 2 5 10 25; do
  FM_UNROLL=$u timeout 300 python bench.py $B --steps 5 > gpurun_out/u_$u.json 2> gpurun_out/u_$u.err
  echo "FM_UNROLL=$u $(python tools/show.py gpurun_out/u_$u.json)" >> gpurun_out/unroll.txt
done
timeout 600 python -m pytest tests -m gpu -x -q -k "run or fullshape" > gpurun_out/pytest_u.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_u.log
echo done
