#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kmeans_tc.py tests/test_gpu_kmeans.py -x -q > gpurun_out/tc2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc2_tests.log
tail -3 gpurun_out/tc2_tests.log
echo "== prefill"; timeout 300 python tools/prefill_jitter.py 5 2>&1 | tail -4
for m in 0 1 2; do
  CKV_TC_MODE=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_assign_tc" -c 4 --csv --log-file gpurun_out/tc2_m$m.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 2 > /dev/null 2>&1
  echo "mode $m: $(grep k_assign_tc gpurun_out/tc2_m$m.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_assign_tc2" --launch-skip 2 -c 1 -o gpurun_out/prof_tc2 -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 3 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q 2>&1 | tail -2
