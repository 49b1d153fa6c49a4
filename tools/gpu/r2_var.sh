#!/bin/bash
# prefill + k_assign_tc2 mode-0 kernel time for the variant libraries named in $VARIANTS
mkdir -p gpurun_out
for v in "" $VARIANTS; do
  if [ -n "$v" ]; then export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_$v.so; else unset CKV_LIB; fi
  P=$(timeout 300 python tools/prefill_jitter.py 4 2>&1 | tail -3 | awk '{print $4}' | tr '\n' ' ')
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_assign_tc" -c 4 --csv --log-file gpurun_out/var_$v.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 2 > /dev/null 2>&1
  echo "[$v] prefill ms: $P | k_assign ns: $(grep k_assign_tc gpurun_out/var_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
