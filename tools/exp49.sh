# deferring trailing lane-qubit ops of store-fix passes to the next pass: A/B in one call
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_parity.py -m gpu -q -x -k "tiled or bench or tile or stale" 2>&1 | tail -1
for w in random30 random28; do
for e in "" "QSB_NO_DEFER_LANE_OPS=1" "" "QSB_NO_DEFER_LANE_OPS=1"; do
  env $e timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$w', '$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'], d['config']['passes'])" || tail -3 gpurun_out/sr.err
done
done
python tools/pass_profile.py --n 30 > gpurun_out/pp_defer.jsonl 2>/dev/null
