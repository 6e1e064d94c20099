# knob sweep on the current code (random30, same call)
for e in "" "QSB_TILE_EARLY=4" "QSB_TILE_EARLY=8" "QSB_NO_WARP_TRANSPOSE=1" "QSB_TILE_R=5" "QSB_FREE_LOAD=0" ""; do
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'], d['config']['passes'])" || tail -3 gpurun_out/sr.err
done
