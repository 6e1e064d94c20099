timeout 900 python -m pytest tests/test_shard_ipc_gpu.py -x -q 2>&1 | tail -25
