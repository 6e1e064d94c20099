python tools/kernel_probe.py --n 28 --reps 5 > gpurun_out/kernel_probe_28.jsonl 2> gpurun_out/kernel_probe_28.err; echo rc=$?
cat gpurun_out/kernel_probe_28.jsonl; tail -5 gpurun_out/kernel_probe_28.err
python tools/kernel_probe.py --n 28 --reps 1 > gpurun_out/kp_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/kernel_probe_28_ncu.csv python tools/kernel_probe.py --n 28 --reps 1 > gpurun_out/kp_ncu.log 2>&1; echo ncu rc=$?
wc -l gpurun_out/kernel_probe_28_ncu.csv
