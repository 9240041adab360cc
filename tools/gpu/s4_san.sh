# compute-sanitizer over the tensor-core kernels (small shapes)
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_vtc.py -x -q -k "tc and (16-200 or 12-301 or 16-2088)" > gpurun_out/s4_san_mem.log 2>&1; echo "rc=$?" >> gpurun_out/s4_san_mem.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_vtc.py -x -q -k "tc and (16-200 or 12-301)" > gpurun_out/s4_san_race.log 2>&1; echo "rc=$?" >> gpurun_out/s4_san_race.log
echo done
