# zero warps (qubits definite through a pass on the warp bits): parity, then qft30 / random30 A/B in one call
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bench_parity.py -m gpu -q -x -k "stale or qft or tiled or bench or beyond or basis" 2>&1 | tail -2
mkdir -p gpurun_out/jdz; QSB_JIT_CACHE=0 QSB_JIT_DUMP=gpurun_out/jdz python tools/pass_profile.py --n 30 --workload qft > gpurun_out/ppq3.jsonl 2>/dev/null
for w in qft30 random30; do
for e in "" "QSB_NO_ZERO_WARPS=1" "" "QSB_NO_ZERO_WARPS=1"; do
  env $e timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$w', '$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'])" || tail -3 gpurun_out/sr.err
done
done
