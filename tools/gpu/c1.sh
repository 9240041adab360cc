# c1 A/B: parity tests that exercise the M = 8 path, then the device-leg bench line
timeout 900 python -m pytest tests -m gpu -x -q -k "vtc or vacc or run or ops or fullshape" > gpurun_out/pytest_c1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c1.log
B="--no-cpu-baseline --no-e2e"
rm -f gpurun_out/c1.txt
for v in "FM_VACC=simt" "FM_VACC=p" $EXTRA; do
  env $v timeout 300 python bench.py $B --steps 5 > gpurun_out/c1_ab.json 2> gpurun_out/c1_ab.err
  echo "$v $(python tools/show.py gpurun_out/c1_ab.json)" >> gpurun_out/c1.txt
done
echo done
