timeout 1200 python -m pytest tests/test_pathsum_gpu.py tests/test_dropin_gpu.py -x -q 2>&1 | tail -25
