#!/bin/bash
# Lagged k-means control read-back: parity tests, prefill A/B vs CKV_KM_LAG=0, timelines
timeout 1200 python -m pytest tests/test_gpu_kmeans.py tests/test_gpu_kmeans_tc.py tests/test_gpu_headline.py tests/test_gpu_shim.py tests/test_gpu_mcr.py -q -x 2>&1 | tail -3
for rep in 1 2 3; do
for v in "" 0; do
  if [ -n "$v" ]; then export CKV_KM_LAG=0; else unset CKV_KM_LAG; fi
  echo "[lag_off=$v] $(timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['prefill']; print(round(p['ms'],2), 'ms', round(p['frac_of_bf16_peak'],3), min(p['ms_all']), max(p['ms_all']), 'step', round(d['ms_per_step']*1000,1))")"
done
done
unset CKV_KM_LAG
timeout 300 python tools/prefill_timeline.py 2>/dev/null | head -3
CKV_KM_OVERLAP=0 timeout 300 python tools/prefill_timeline.py 2>/dev/null | head -3
