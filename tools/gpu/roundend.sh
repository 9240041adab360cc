# What the driver runs at round end (one B200): GPU tests, smoke, the default bench and the reference arm
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/re_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/re_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/re_smoke.log
timeout 900 python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err; echo "rc=$?" >> gpurun_out/re_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/re_ref.json 2> gpurun_out/re_ref.err; echo "rc=$?" >> gpurun_out/re_ref.err
echo done
