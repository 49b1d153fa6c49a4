#!/bin/bash
# k_attend guided tail (finer splits for the last q heads of the counter schedule)
timeout 900 python -m pytest tests/test_gpu_attend.py tests/test_gpu_session.py tests/test_gpu_headline.py tests/test_gpu_sharded_decode.py tests/test_gpu_select.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for v in "8 4" "0 4" "4 4" "8 8" "16 4" "4 2"; do
  set -- $v
  echo "[div=$1 mul=$2] $(CKV_AT_TAIL_DIV=$1 CKV_AT_TAIL_SPLIT=$2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 3 --no-cpu --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step']*1000,2), 'attend', round(d['roofline']['launch_us'],1), 'frac', round(d['roofline']['frac'],3))")"
done
done
