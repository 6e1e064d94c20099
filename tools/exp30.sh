timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py tests/test_bench_parity.py tests/test_dropin_gpu.py -m gpu -q -x 2>&1 | tail -3
python tools/scan_probe.py --n 28
timeout 600 python tools/kernel_probe.py --n 28 > gpurun_out/kp28f.jsonl 2> gpurun_out/kp28f.err; echo kp rc=$?
