#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_kmeans_tc.py tests/test_gpu_kmeans.py -x -q 2>&1 | tail -1 > gpurun_out/t.log; cat gpurun_out/t.log
export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_prof.so
timeout 300 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 2 2>&1 | grep t2prof | head -1
unset CKV_LIB
VARIANTS="" bash tools/gpu/r2_var.sh
