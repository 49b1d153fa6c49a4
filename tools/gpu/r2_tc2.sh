#!/bin/bash
# k_assign_tc2 check: k-means parity tests, prefill timing v2 vs v1, per-mode kernel times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kmeans_tc.py tests/test_gpu_kmeans.py tests/test_gpu_headline.py -x -q > gpurun_out/tc2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc2_tests.log
tail -3 gpurun_out/tc2_tests.log
echo "== v2"; timeout 300 python tools/prefill_jitter.py 6 2>&1 | tail -6
echo "== v1"; CKV_TC_V1=1 timeout 300 python tools/prefill_jitter.py 4 2>&1 | tail -4
for m in 0 1 2; do
CKV_TC_MODE=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_assign_tc" --csv --log-file gpurun_out/tc2_mode$m.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 2 > /dev/null 2>&1
echo "mode $m: $(grep k_assign_tc gpurun_out/tc2_mode$m.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
