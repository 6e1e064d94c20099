# flip frame on/off, alternating in one call (second box)
for e in "" "QSB_NO_FLIP_FRAME=1" "" "QSB_NO_FLIP_FRAME=1" "" "QSB_NO_FLIP_FRAME=1"; do
  env $e timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'])" || tail -3 gpurun_out/sr.err
done
