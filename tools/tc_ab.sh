# A/B of k_assign_tc launch time (ncu, serialised) for the product library
# and the libraries named in $VARIANTS (tools/build_variant.py), config B.
for v in "" $VARIANTS; do
  if [ -n "$v" ]; then export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_$v.so; else unset CKV_LIB; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KREGEX:-k_assign_tc|k_fixup}" --csv \
      --log-file gpurun_out/tc_ab_$v.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 \
      --no-cpu --no-extra --max-iters 3 > /dev/null 2>&1
  echo "[$v]"; python tools/launch_table.py gpurun_out/tc_ab_$v.csv | head -3
done
