timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py tests/test_bench_parity.py -q -x 2>&1 | tail -3
python tools/kernel_probe.py --n 28 --reps 5 > gpurun_out/kernel_probe_28d.jsonl 2> gpurun_out/kernel_probe_28d.err; echo rc=$?
cut -c1-130 gpurun_out/kernel_probe_28d.jsonl
python tools/kernel_probe.py --n 28 --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/kernel_probe_28d_ncu.csv python tools/kernel_probe.py --n 28 --reps 1 > /dev/null 2>&1; echo ncu rc=$?
