timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_kernels or custom or per_gate" 2>&1 | tail -3
python tools/kernel_probe.py --n 28 --reps 5 2>/dev/null | grep -E "dense|flip" | cut -c1-120
