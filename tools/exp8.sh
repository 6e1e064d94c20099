export QSB_BENCH_PASSES=1
for v in "QSB_TILE_R=4" "QSB_TILE_R=5" "QSB_TILE_R=0"; do
  env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}.json 2>/dev/null
done
