QSB_STORE_KEEP=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tiled or tile or bench" 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -12
QSB_STORE_KEEP=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tiled or tile or bench" 2>&1 | tail -1
for e in "" "QSB_STORE_KEEP=2" "QSB_STORE_KEEP=3" "" "QSB_STORE_KEEP=2" "QSB_STORE_KEEP=3"; do
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'], d['config']['passes'])"
done
QSB_STORE_KEEP=2 python tools/pass_profile.py --n 30 > gpurun_out/pass_profile_k2.jsonl 2>/dev/null
