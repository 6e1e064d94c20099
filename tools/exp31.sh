timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py -m gpu -q -x -k "scan or cumulative or serial or sample or counts or sweep or bitwise" 2>&1 | tail -3
python tools/scan_probe.py --n 28
timeout 600 python tools/kernel_probe.py --n 28 > gpurun_out/kp28g.jsonl 2> gpurun_out/kp28g.err; echo kp rc=$?
