#!/bin/bash
# racecheck: the session steps (StepSync, decode-batch k-means) and the
# decode-batch suite, clustered selection path off (racecheck does not model
# DSMEM stores)
O=gpurun_out; mkdir -p $O
for t in test_gpu_session test_gpu_decode_batch; do
  CKV_SEL_NC=1 timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/$t.py -x -q > $O/race_${t}_nc1.txt 2>&1
  echo "racecheck $t (NC=1): $(grep 'RACECHECK SUMMARY' $O/race_${t}_nc1.txt | tail -1) | $(grep -E 'passed|failed' $O/race_${t}_nc1.txt | tail -1)"
done
timeout 600 python -m pytest tests/test_gpu_decode_batch.py tests/test_gpu_session.py -m gpu -x -q 2>&1 | tail -1
