# A/B of the current library against build/old/libfastmnmf.so (an older commit built by hand) on one box
L=paper_1903_03237_b200/libfastmnmf.so
cp $L /tmp/new.so
rm -f gpurun_out/ab_old.txt
for c in c2 c3 c1; do
  B="--config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  for v in new old; do
    if [ $v = old ]; then cp build/old/libfastmnmf.so $L; else cp /tmp/new.so $L; fi
    timeout 600 python bench.py $B > gpurun_out/ab_${c}_$v.json 2> gpurun_out/ab_${c}_$v.err
    echo "$c $v $(python tools/show.py gpurun_out/ab_${c}_$v.json)" >> gpurun_out/ab_old.txt
  done
done
cp /tmp/new.so $L
echo done
