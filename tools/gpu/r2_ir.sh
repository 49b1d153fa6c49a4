#!/bin/bash
# attention item size under the dynamic schedule
mkdir -p gpurun_out
run() {
  timeout -k 10 300 python bench.py --steps 50 --warmup 10 --e2e-steps 20 --no-cpu --no-extra --max-iters 8 > gpurun_out/ir.json 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/ir.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$1', 'us/step', round(d.get('ms_per_step')*1000,1), 'e2e us', round(1e6/d['e2e']['value'],1), 'layer us', round(d['per_layer']['ms_per_step']*1000,1))"
}
for r in 1 2; do
  for v in "" s3 t32s4 t32s3; do
    if [ -n "$v" ]; then export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_$v.so; else unset CKV_LIB; fi
    run "ir${v:-1024}"
  done
done
