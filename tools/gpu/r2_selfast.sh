#!/bin/bash
# selection: bulk-copy centroid ring with L2 hints; step time and phases
mkdir -p gpurun_out
timeout -k 10 500 python -m pytest tests/test_gpu_select.py tests/test_gpu_session.py tests/test_gpu_headline.py tests/test_gpu_attend.py -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do
  timeout -k 10 300 python bench.py --steps 50 --warmup 10 --e2e-steps 20 --no-cpu --no-extra --max-iters 8 > gpurun_out/selfast.json 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/selfast.json'):
    if l.startswith('{'):
        d=json.loads(l); print('ms/step', d.get('ms_per_step'), 'value', d.get('value'), 'e2e', (d.get('e2e') or {}).get('value'))"
done
export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_seldbg.so
echo "persist on:"; CKV_DEBUG_TIMING=1 timeout 300 python bench.py --steps 4 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 4 2>&1 | grep "k_select_fused dbg" | tail -3
