# qft30 (12-qubit tiles): register bits 3 / 4 / 5 for every pass, same call
for e in "" "QSB_TILE_R=3" "QSB_TILE_R=5" "" "QSB_TILE_R=3"; do
  env $e timeout 600 python bench.py --workload qft30 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$e', d['value'], d['ms_per_step'], d['parity']['ok'])" || tail -2 gpurun_out/sr.err
done
