timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py tests/test_pathsum_gpu.py tests/test_dropin_gpu.py -q -x 2>&1 | tail -3
python tools/kernel_probe.py --n 28 --reps 5 > gpurun_out/kernel_probe_28f.jsonl 2>/dev/null; cut -c1-110 gpurun_out/kernel_probe_28f.jsonl | head -12; grep pauli gpurun_out/kernel_probe_28f.jsonl | cut -c1-120
