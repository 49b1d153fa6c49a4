#!/bin/bash
# attention: item metadata loaded one item ahead, item descriptors to the consumers
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_gpu_attend.py tests/test_gpu_session.py tests/test_gpu_headline.py tests/test_gpu_sharded_decode.py tests/test_gpu_page.py tests/test_gpu_metrics.py -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do
  timeout -k 10 300 python bench.py --steps 50 --warmup 10 --e2e-steps 20 --no-cpu --no-extra --max-iters 8 > gpurun_out/ahead.json 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/ahead.json'):
    if l.startswith('{'):
        d=json.loads(l); print('us/step', round(d.get('ms_per_step')*1000,1), 'e2e us', round(1e6/d['e2e']['value'],1), 'layer us', round(d['per_layer']['ms_per_step']*1000,1), 'attend us', round(d['kernels_us']['k_attend'],1), 'frac', round(d['roofline']['frac'],3))"
done
