#!/bin/bash
CKV_TRACE_HOST=1 timeout 600 python tools/prefill_jitter.py 14 > gpurun_out/jit.out 2> gpurun_out/jit.err
cat gpurun_out/jit.out
