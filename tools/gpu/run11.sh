timeout 900 python -m pytest tests/test_gpu_session.py -x -q -k "tier" 2>&1 | tail -15
