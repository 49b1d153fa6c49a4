# A/B prefill timing: product library vs the libraries named in $VARIANTS
# (built by tools/build_variant.py), alternating, config B.
for rep in 1 2; do
for v in "" $VARIANTS; do
  if [ -n "$v" ]; then export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_$v.so; else unset CKV_LIB; fi
  echo "[$v] $(python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['prefill']; print(round(p['ms'],2), 'ms', round(p['frac_of_bf16_peak'],3), 'step', round(d['ms_per_step']*1000,1))")"
done
done
