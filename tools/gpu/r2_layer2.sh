#!/bin/bash
# layer mode with StepSync on the split selection path
mkdir -p gpurun_out
timeout -k 10 500 python -m pytest tests/test_gpu_session.py tests/test_gpu_headline.py tests/test_gpu_select.py -m gpu -x -q 2>&1 | tail -2
for v in on off on off; do
  if [ $v = off ]; then export CKV_SESSION_NO_STEPSYNC=1; else unset CKV_SESSION_NO_STEPSYNC; fi
  echo "stepsync $v: $(timeout -k 10 300 python tools/layer_prof.py 20 8 2>&1 | tail -3 | tr '\n' ' ')"
done
