python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_plain.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_random30_r2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1; echo rc=$?
python bench.py --workload qft30 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_plain.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_qft30_r2.csv python bench.py --workload qft30 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_ncu.log 2>&1; echo rc=$?
