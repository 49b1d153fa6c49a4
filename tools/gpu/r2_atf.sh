#!/bin/bash
# FFMA2 in the attention's logits / value update: parity + step A/B
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_attend.py tests/test_gpu_session.py -m gpu -x -q 2>&1 | tail -2
B="python bench.py --steps 50 --warmup 10 --e2e-steps 10 --no-cpu --no-extra --max-iters 8"
show() { python -c "
import json,sys
for l in open('gpurun_out/sp.json'):
    if l.startswith('{'):
        d=json.loads(l); pl=d.get('per_layer') or {}; print('$1', 'us/step', round(d['ms_per_step']*1000,1), 'sel', round(d['kernels_us']['k_select'],1), 'att', round(d['kernels_us']['k_attend'],1), 'e2e', round(d['e2e']['value']), 'layer_ms', round(pl.get('ms_per_step'),4))"; }
for r in 1 2 3; do
timeout 300 $B > gpurun_out/sp.json 2>gpurun_out/sp.err; show ffma2
CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_atfma.so timeout 300 $B > gpurun_out/sp.json 2>/dev/null; show fma
done
