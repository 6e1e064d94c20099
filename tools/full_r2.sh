# full GPU validation + measurements (round 2)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? ; tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
python bench.py --workload qft30 --steps 10 > gpurun_out/bench_qft30.json 2> gpurun_out/bench_qft30.err; echo qft rc=$?
python bench.py --workload random28 --steps 10 --no-cpu-baseline > gpurun_out/bench_random28.json 2> gpurun_out/bench_random28.err; echo r28 rc=$?
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref rc=$?
cat gpurun_out/bench_default.json gpurun_out/bench_qft30.json gpurun_out/bench_random28.json gpurun_out/bench_reference.json | cut -c1-400
