timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py tests/test_dropin_gpu.py -x -q 2>&1 | tail -8
python tools/kernel_probe.py --n 28 --reps 5 > gpurun_out/kernel_probe_28b.jsonl 2> gpurun_out/kernel_probe_28b.err; echo rc=$?
cat gpurun_out/kernel_probe_28b.jsonl | cut -c1-150; tail -3 gpurun_out/kernel_probe_28b.err
