timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense or pair or per_gate" 2>&1 | tail -2
timeout 600 python tools/kernel_probe.py --n 28 > gpurun_out/kp28c.jsonl 2> gpurun_out/kp28c.err; echo kp rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/kp28c_ncu.csv python tools/kernel_probe.py --n 28 --reps 1 > gpurun_out/kp28c_ncu.log 2>&1; echo ncu rc=$?
