# final ncu evidence: per-kernel DRAM launch list of the kernel probe, ncu --set full of random30 passes 0-5
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/kp28_ncu_final.csv python tools/kernel_probe.py --n 28 --reps 1 > gpurun_out/kp28_ncu_final.log 2>&1; echo kp-ncu rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qsb_tile -s 0 -c 6 -o gpurun_out/r2f_random30_passes0-5 python tools/prof_run.py --n 30 --reps 1 > gpurun_out/prof_ncu_final.log 2>&1; echo full rc=$?
