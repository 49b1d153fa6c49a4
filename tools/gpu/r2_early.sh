#!/bin/bash
# the selection streaming its centroids before its grid dependency wait
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_gpu_session.py tests/test_gpu_headline.py tests/test_gpu_quality.py tests/test_gpu_trace.py -m gpu -x -q 2>&1 | tail -1
run() {
  timeout -k 10 300 python bench.py --steps 50 --warmup 10 --e2e-steps 20 --no-cpu --no-extra --max-iters 8 > gpurun_out/early.json 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/early.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$1', 'us/step', round(d.get('ms_per_step')*1000,1), 'e2e us', round(1e6/d['e2e']['value'],1), 'layer us', round(d['per_layer']['ms_per_step']*1000,1))"
}
for r in 1 2; do
  unset CKV_SESSION_NO_EARLY; run early
  CKV_SESSION_NO_EARLY=1 run noearly
done
