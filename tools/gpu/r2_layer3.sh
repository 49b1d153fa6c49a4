#!/bin/bash
# layer mode: clustered fused selection (default for few units) vs split K1 + K2
mkdir -p gpurun_out
timeout -k 10 500 python -m pytest tests/test_gpu_select.py tests/test_gpu_session.py tests/test_gpu_headline.py tests/test_gpu_quality.py tests/test_gpu_trace.py -m gpu -x -q 2>&1 | tail -3
for v in def few def few; do
  if [ $v = few ]; then export CKV_SEL_FEW=1; else unset CKV_SEL_FEW; fi
  echo "$v: $(timeout -k 10 300 python tools/layer_prof.py 20 8 2>&1 | tail -3 | tr '\n' ' ')"
done
for n in 2 4; do echo "NC=$n: $(CKV_SEL_NC=$n timeout -k 10 300 python tools/layer_prof.py 20 8 2>&1 | tail -1)"; done
