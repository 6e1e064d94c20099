timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py -q -x -k "sample or cumulative or serial or pauli or expect or Expectation or count" 2>&1 | tail -3
python tools/kernel_probe.py --n 28 --reps 5 2>/dev/null | grep -E "pauli|sampler|serial|marginal"
python bench.py --force-dist --config4-qubits 26 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_forcedist.json 2> gpurun_out/bench_forcedist.err; echo fd rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_forcedist.json')); print(d['value'], d['config']['parallelism'], json.dumps(d.get('config4')))"; tail -3 gpurun_out/bench_forcedist.err
python tools/prof_run.py --n 30 --reps 1 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qsb_tile -s 0 -c 6 -o gpurun_out/r2_random30_passes0-5 python tools/prof_run.py --n 30 --reps 1 > gpurun_out/prof_ncu.log 2>&1; echo ncu rc=$?
