#!/bin/bash
# e2e: q by the copy engine (default) vs zero-copy q reads (CKV_SESSION_Q_ZC=1)
timeout 900 python -m pytest tests/test_gpu_session.py tests/test_gpu_headline.py -q -x 2>&1 | tail -2
for rep in 1 2 3; do
for v in "" 1; do
  if [ -n "$v" ]; then export CKV_SESSION_Q_ZC=1; else unset CKV_SESSION_Q_ZC; fi
  echo "[q_zc=$v] $(timeout 300 python bench.py --steps 10 --warmup 5 --e2e-steps 30 --no-cpu --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step']*1000,2), 'e2e us', round(1e6/d['e2e']['value'],1))")"
done
done
unset CKV_SESSION_Q_ZC
timeout 300 python tools/e2e_timeline.py 4 > gpurun_out/e2e_tl3.txt 2>&1; head -1 gpurun_out/e2e_tl3.txt; tail -12 gpurun_out/e2e_tl3.txt
