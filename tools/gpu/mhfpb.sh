B="--no-cpu-baseline --no-e2e --config c4mh --steps 3 --warmup 3"
for v in 1 2 4; do FM_MH_FPB=$v timeout 300 python bench.py $B > gpurun_out/mh_fpb$v.json 2>> gpurun_out/mhfpb.err; done
echo done
