timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py tests/test_dropin_gpu.py -x -q -k "expect or pauli or marginal or prob or dense or custom or sample or gradient or Expectation or Gradient" 2>&1 | tail -4
python tools/kernel_probe.py --n 28 --reps 5 > gpurun_out/kernel_probe_28c.jsonl 2> gpurun_out/kernel_probe_28c.err; echo rc=$?
cat gpurun_out/kernel_probe_28c.jsonl | cut -c1-120; tail -3 gpurun_out/kernel_probe_28c.err
