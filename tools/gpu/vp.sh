# k_vacc_p (persistent V accumulation) at c1: parity tests, then chunk size x CTAs per SM
timeout 900 python -m pytest tests/test_gpu_vtc.py -x -q -k persistent > gpurun_out/pytest_vp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_vp.log
B="--no-cpu-baseline --no-e2e"
rm -f gpurun_out/vp.txt
for v in "FM_VACC=simt" "FM_VACC=p FM_VP_TB=256 FM_VP_CTAS=3" "FM_VACC=p FM_VP_TB=256 FM_VP_CTAS=2" "FM_VACC=p FM_VP_TB=128 FM_VP_CTAS=4" "FM_VACC=p FM_VP_TB=128 FM_VP_CTAS=3" "FM_VACC=p FM_VP_TB=128 FM_VP_CTAS=2"; do
  env $v timeout 300 python bench.py $B --steps 5 > gpurun_out/vp1.json 2> gpurun_out/vp1.err
  echo "$v $(python tools/show.py gpurun_out/vp1.json)" >> gpurun_out/vp.txt
done
echo done
