python -m pytest tests/test_bench_parity.py tests/test_gpu_parity.py -x -q -k "bench_path or sharded_p8 or serial_checksum" 2>&1 | tail -15
python bench.py --workload qft30 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_qft30.json 2> gpurun_out/bench_qft30.err
cat gpurun_out/bench_qft30.json; tail -3 gpurun_out/bench_qft30.err
