timeout 900 python -m pytest tests/test_gpu_quality.py tests/test_gpu_metrics.py -x -q 2>&1 | tail -25
