#!/bin/bash
# sanitizer pass over the kernels changed after the closing evidence
O=gpurun_out; mkdir -p $O
for t in test_gpu_attend test_gpu_session test_gpu_kmeans_tc test_gpu_select; do
  timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/$t.py -x -q > $O/san2_$t.txt 2>&1
  echo "memcheck $t: $(grep 'ERROR SUMMARY' $O/san2_$t.txt | tail -1) | $(grep -E 'passed|failed' $O/san2_$t.txt | tail -1)"
done
for t in test_gpu_attend test_gpu_session; do
  CKV_SEL_NC=1 timeout 1500 compute-sanitizer --tool racecheck python -m pytest tests/$t.py -x -q > $O/race2_$t.txt 2>&1
  echo "racecheck $t (NC=1): $(grep 'RACECHECK SUMMARY' $O/race2_$t.txt | tail -1) | $(grep -E 'passed|failed' $O/race2_$t.txt | tail -1)"
done
