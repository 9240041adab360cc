# k_vacc_blk: parity tests, then c1/c2/c3 bench lines for the default vs the previous kernels
timeout 900 python -m pytest tests/test_gpu_vtc.py tests/test_gpu_run.py tests/test_gpu_dp.py -x -q > gpurun_out/pytest_vblk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_vblk.log
B="--no-cpu-baseline --no-e2e"
timeout 300 python bench.py $B --steps 5 > gpurun_out/c1_blk.json 2> gpurun_out/c1_blk.err
timeout 300 python bench.py $B --config c3 --steps 2 --warmup 3 --iters 20 > gpurun_out/c3_blk.json 2> gpurun_out/c3_blk.err
timeout 600 python bench.py $B --config c2 --steps 3 --warmup 3 > gpurun_out/c2_blk.json 2> gpurun_out/c2_blk.err
FM_VACC=blk timeout 600 python bench.py $B --config c2 --steps 3 --warmup 3 > gpurun_out/c2_blkf.json 2>> gpurun_out/c2_blk.err
timeout 300 python bench.py $B --config c4 --steps 3 --warmup 3 > gpurun_out/c4_blk.json 2> gpurun_out/c4_blk.err
echo done
