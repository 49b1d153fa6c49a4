#!/bin/bash
# Append folded into the fused selection: session parity tests, then e2e A/B
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_session.py tests/test_gpu_headline.py tests/test_gpu_trace.py tests/test_gpu_quality.py -q -x 2>&1 | tail -3
for rep in 1 2 3; do
for v in "" 1; do
  if [ -n "$v" ]; then export CKV_SESSION_NO_FOLD_APPEND=1; else unset CKV_SESSION_NO_FOLD_APPEND; fi
  echo "[nofold=$v] $(timeout 300 python bench.py --no-extra --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step']*1000,2), 'e2e', round(1e6/d['e2e']['value'],1), d['per_layer']['us_per_layer'] if d.get('per_layer') else '')")"
done
done
unset CKV_SESSION_NO_FOLD_APPEND
timeout 300 python tools/e2e_timeline.py 4 > $O/e2e_tl2.txt 2>&1; tail -40 $O/e2e_tl2.txt
