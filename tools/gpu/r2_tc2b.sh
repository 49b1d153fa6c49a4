#!/bin/bash
# chunk-width variants of k_assign_tc2: prefill time, per-mode kernel time; one full ncu capture
mkdir -p gpurun_out
for v in "" cw256 cw64; do
  if [ -n "$v" ]; then export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_$v.so; else unset CKV_LIB; fi
  echo "== [$v] prefill"; timeout 300 python tools/prefill_jitter.py 4 2>&1 | tail -3
  for m in 0 2; do
    CKV_TC_MODE=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_assign_tc" -c 4 --csv --log-file gpurun_out/tc2_$v$m.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 2 > /dev/null 2>&1
    echo "mode $m: $(grep k_assign_tc gpurun_out/tc2_$v$m.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
  done
done
unset CKV_LIB
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_assign_tc2" --launch-skip 2 -c 1 -o gpurun_out/prof_tc2 -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 3 > /dev/null 2>&1
ls -la gpurun_out/prof_tc2.ncu-rep
