timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bench_parity.py tests/test_shard_gpu.py tests/test_pathsum_gpu.py -m gpu -q -x 2>&1 | tail -2
for e in "" "QSB_NO_FLIP_FRAME=1" "" "QSB_NO_FLIP_FRAME=1"; do
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'], d['config']['passes'])"
done
python tools/pass_profile.py --n 30 > gpurun_out/pass_profile_frame.jsonl 2>/dev/null
