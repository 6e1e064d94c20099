python tools/scan_probe.py --n 28
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/scan_ncu.csv python tools/scan_probe.py --n 28 --reps 1 > gpurun_out/scan_ncu.log 2>&1; echo ncu rc=$?
