# new register-width costs (R5 preferred unless it needs more exchanges): random30 and random28, same call
for w in random30 random28; do
for e in "" "QSB_TILE_R=5" "QSB_TILE_R=4" "" "QSB_TILE_R=5"; do
  env $e timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$w', '$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'])" || tail -3 gpurun_out/sr.err
done
done
