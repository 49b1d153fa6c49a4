#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_session.py tests/test_gpu_trace.py tests/test_gpu_headline.py tests/test_gpu_quality.py tests/test_gpu_shim.py -x -q 2>&1 | tail -2
timeout 600 python tools/layer_prof.py 20 8
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_attend" -c 12 --csv --log-file gpurun_out/b_launch.csv python tools/layer_prof.py 3 8 > /dev/null 2>&1
grep -E "k_select|k_attend" gpurun_out/b_launch.csv | awk -F'","' '{print substr($5,1,30), $NF}' | head -12
