# full GPU tests + the c1 / c2 / c3 device-leg bench lines
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
B="--no-cpu-baseline --no-e2e"
rm -f gpurun_out/c123.txt
timeout 300 python bench.py $B --steps 5 > gpurun_out/t_c1.json 2> gpurun_out/t_c1.err
timeout 300 python bench.py $B --config c3 --steps 2 --warmup 3 --iters 20 > gpurun_out/t_c3.json 2> gpurun_out/t_c3.err
timeout 600 python bench.py $B --config c2 --steps 3 --warmup 3 > gpurun_out/t_c2.json 2> gpurun_out/t_c2.err
python tools/show.py gpurun_out/t_c1.json gpurun_out/t_c2.json gpurun_out/t_c3.json > gpurun_out/c123.txt
echo done
