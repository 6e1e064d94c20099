for e in "" "QSB_TILE_SINGLEBUF=1" "QSB_TILE_MINB=2" "QSB_TILE_MINB=3 QSB_TILE_SINGLEBUF=1" "QSB_TILE_MINB=2 QSB_TILE_SINGLEBUF=1" ""; do
  env $e timeout 600 python bench.py --workload qft30 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q.json 2>gpurun_out/q.err
  python -c "import json; d=json.load(open('gpurun_out/q.json')); print('$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'])" || tail -3 gpurun_out/q.err
done
