#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 400 python -m pytest tests/test_gpu_kmeans_tc.py tests/test_gpu_kmeans.py tests/test_gpu_headline.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do
for v in "" ff4; do
  if [ -n "$v" ]; then export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_$v.so; else unset CKV_LIB; fi
  echo "[${v:-ff16}] prefill ms: $(timeout -k 10 150 python tools/prefill_jitter.py 4 2>&1 | tail -3 | awk '{print $4}' | tr '\n' ' ')"
done
done
unset CKV_LIB
timeout -k 10 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fixup_full" -c 12 --csv --log-file gpurun_out/ff.csv python tools/prefill_jitter.py 1 > /dev/null 2>&1
echo "k_fixup_full ns: $(grep k_fixup_full gpurun_out/ff.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
