timeout 600 python -m pytest tests/test_gpu_kmeans_tc.py tests/test_gpu_kmeans.py tests/test_gpu_mcr.py -x -q 2>&1 | tail -5
timeout 300 python tools/prefill_jitter.py 6 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -5
ncu --set full --import-source on --clock-control none -k regex:k_assign_tc -s 10 -c 1 -o gpurun_out/assign_r2c python tools/prefill_jitter.py 1 > /dev/null 2>&1
