#!/bin/bash
# host submit cost and e2e after trimming per-launch host work
mkdir -p gpurun_out
timeout -k 10 300 python tools/host_overhead.py 2>&1 | tail -4
for r in 1 2; do
  timeout -k 10 300 python bench.py --steps 30 --warmup 5 --e2e-steps 60 --no-cpu --no-extra --max-iters 8 > gpurun_out/e2e.json 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/e2e.json'):
    if l.startswith('{'):
        d=json.loads(l); print('ms/step', round(d.get('ms_per_step')*1000,1), 'e2e tok/s', round(d['e2e']['value']), 'e2e us', round(1e6/d['e2e']['value'],1))"
done
