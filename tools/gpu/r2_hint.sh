#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
for v in "" nohint; do
  if [ -n "$v" ]; then export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_$v.so; else unset CKV_LIB; fi
  timeout -k 10 300 python bench.py --steps 50 --warmup 10 --e2e-steps 10 --no-cpu --no-extra --max-iters 8 > gpurun_out/hint.json 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/hint.json'):
    if l.startswith('{'):
        d=json.loads(l); print('${v:-hint}', 'us/step', round(d.get('ms_per_step')*1000,1), 'attend us', round(d['kernels_us']['k_attend'],1), 'select us', round(d['kernels_us']['k_select'],1))"
done
done
