export QSB_BENCH_PASSES=1
for v in "" "QSB_TILE_EARLY=8" "QSB_TILE_EARLY=12" "QSB_TILE_R=5"; do
  env $v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pp_${v:-default}.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pp_${v:-default}.json')); r=d['roofline']
print('${v:-default}', d['value'], d['ms_per_step'], r['frac'], r['launch_ms'])"
done
