export QSB_JIT_DEBUG=1
python bench.py --workload qft30 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_qft30b.json 2> gpurun_out/bench_qft30b.err
cat gpurun_out/bench_qft30b.json | python -c "import json,sys; d=json.load(sys.stdin); print(json.dumps(d['e2e']['cold'], indent=1))"
grep -c "disk" gpurun_out/bench_qft30b.err; head -30 gpurun_out/bench_qft30b.err
