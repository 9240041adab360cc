timeout 900 python tools/fullrank_bench.py > gpurun_out/fullrank_bench.jsonl 2> gpurun_out/fullrank_bench.err
timeout 300 python tools/stft_bench.py > gpurun_out/stft_bench.txt 2> gpurun_out/stft_bench.err
echo done
