#!/bin/bash
# summarise gpurun_out/bench_*.json and the launch list
cd /root/repo
for c in "$@"; do python -c "
import json,sys
try:
  d=json.load(open('gpurun_out/bench_$c.json'))
except Exception as e:
  print('$c', 'ERR', open('gpurun_out/bench_$c.err').read()[-1500:]); sys.exit()
r=d['roofline']; print('$c', 'it/s %.1f'%d['iters_per_s'], 'val %.3g'%d['value'], 'frac %.3f'%r['frac'], r['kernel'], {k:round(v*1000,1) for k,v in r['kernel_ms'].items()}, 'e2e', d['e2e'] and '%.3g'%d['e2e']['value'], d['clocks'])
"; done
