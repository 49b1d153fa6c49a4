# A/B of the config B decode step: product library vs $VARIANTS (tools/build_variant.py)
for rep in 1 2 3; do
for v in "" $VARIANTS; do
  if [ -n "$v" ]; then export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_$v.so; else unset CKV_LIB; fi
  echo "[$v] $(python bench.py --no-extra --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step']*1000,2), d['kernels_us'])")"
done
done
