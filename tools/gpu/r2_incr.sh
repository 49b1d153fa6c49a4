#!/bin/bash
# prefill: incremental centroid update from pass N (CKV_KM_INCR_FROM)
mkdir -p gpurun_out
timeout -k 10 400 python -m pytest tests/test_gpu_kmeans_tc.py tests/test_gpu_kmeans.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do
for v in 5 2 3 4; do
  echo "INCR_FROM=$v: $(CKV_KM_INCR_FROM=$v timeout -k 10 150 python tools/prefill_jitter.py 4 2>&1 | tail -3 | awk '{print $4}' | tr '\n' ' ')"
done
done
