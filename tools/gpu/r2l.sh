timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2l.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2l.log
timeout 600 python bench.py --config c3 --shard --steps 2 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e > gpurun_out/r2l_c3shard.json 2> gpurun_out/r2l_c3shard.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --iters 20 > gpurun_out/r2l_torchrun.json 2> gpurun_out/r2l_torchrun.err
echo done
