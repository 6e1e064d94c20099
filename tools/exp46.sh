timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bench_parity.py tests/test_dropin_gpu.py tests/test_cli_gpu.py tests/test_pathsum_gpu.py -m gpu -q -x 2>&1 | tail -1
for w in qft30 random30; do
for e in "" "QSB_NO_ZERO_STORE_SKIP=1" "" "QSB_NO_ZERO_STORE_SKIP=1"; do
  env $e timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$w', '$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'])" || tail -3 gpurun_out/sr.err
done
done
python tools/pass_profile.py --n 30 --workload qft > gpurun_out/ppq2.jsonl 2>/dev/null
