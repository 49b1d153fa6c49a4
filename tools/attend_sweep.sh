#!/bin/bash
# k_attend tile / stage / item-size sweep over experiment builds
# (tools/build_variant.py ckv_attend.cu <tag> -D...); config B bench.
for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then L=""; else L=paper_2412_03213_b200/libckv_b200_$v.so; fi
  for rep in 1 2; do
  CKV_LIB=$L python bench.py --no-cpu --no-extra --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['select_attend_us_per_step'],1), {k: round(v,1) for k,v in d['kernels_us'].items()}, round(d['roofline']['frac'],3), round(d['step_roofline']['frac'],3))"
  done
done
