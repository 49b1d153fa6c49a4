#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_kmeans_tc.py tests/test_gpu_kmeans.py tests/test_gpu_headline.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_assign_tc2" --launch-skip 2 -c 1 -o gpurun_out/prof_tc2 -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 3 > /dev/null 2>&1
ls -la gpurun_out/prof_tc2.ncu-rep
