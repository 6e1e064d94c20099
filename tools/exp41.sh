# per-pass register width choice vs 5 register bits everywhere (alternating, same call)
for e in "" "QSB_TILE_R=5" "" "QSB_TILE_R=5" "" "QSB_TILE_R=5"; do
  env $e timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'])" || tail -3 gpurun_out/sr.err
done
