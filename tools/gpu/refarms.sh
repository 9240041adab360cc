# The reference arm (numpy restatement on the box's host cores) for the other configs
for c in c2 c4 c4mh; do
  timeout 900 python bench.py --impl reference --config $c --steps 2 --warmup 3 > gpurun_out/ref_$c.json 2> gpurun_out/ref_$c.err
done
timeout 1500 python bench.py --impl reference --config c3 --steps 1 --warmup 3 > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err
echo done
