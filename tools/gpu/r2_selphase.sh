#!/bin/bash
# selection phases in the batched step: step time, scoring-only mode, per-head stamps
mkdir -p gpurun_out
B="python bench.py --steps 50 --warmup 10 --e2e-steps 10 --no-cpu --no-extra --max-iters 8"
show() { python -c "
import json,sys
for l in open('gpurun_out/sp.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$1', 'us/step', round(d['ms_per_step']*1000,1), 'sel', round(d['kernels_us']['k_select'],1), 'att', round(d['kernels_us']['k_attend'],1), 'e2e', round(d['e2e']['value']))"; }
timeout 300 $B > gpurun_out/sp.json 2>/dev/null; show base
CKV_SEL_MODE=1 timeout 300 $B > gpurun_out/sp.json 2>/dev/null; show score_only
export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_seldbg.so
CKV_DEBUG_TIMING=1 timeout 300 python bench.py --steps 4 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 4 2>&1 | grep "k_select_fused dbg" | tail -3
