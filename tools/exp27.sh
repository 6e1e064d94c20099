timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cli_gpu.py tests/test_dropin_gpu.py tests/test_shard_gpu.py -m gpu -q -x 2>&1 | tail -2
timeout 600 python tools/kernel_probe.py --n 28 > gpurun_out/kp28d.jsonl 2> gpurun_out/kp28d.err; echo kp rc=$?
