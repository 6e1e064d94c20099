set -x
python -m pytest tests/test_bench_parity.py -x -q 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
tail -3 gpurun_out/bench_r2a.err
cat gpurun_out/bench_r2a.json
