timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py -q -x -k "expect or pauli or Expectation or dense or custom or marginal or prob" 2>&1 | tail -2
python tools/kernel_probe.py --n 28 --reps 5 > gpurun_out/kernel_probe_28e.jsonl 2> gpurun_out/kernel_probe_28e.err; echo rc=$?
cut -c1-110 gpurun_out/kernel_probe_28e.jsonl
python tools/kernel_probe.py --n 28 --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/kernel_probe_28e_ncu.csv python tools/kernel_probe.py --n 28 --reps 1 > /dev/null 2>&1; echo ncu rc=$?
