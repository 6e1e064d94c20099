#!/bin/bash
# Sweeps tile-kernel knobs with bench.py (values only).  Usage: tools/sweep.sh <workload>
W=${1:-random30}
for cfg in "QSB_TILE_PREFETCH=0 QSB_TILE_M=12" "QSB_TILE_PREFETCH=1 QSB_TILE_M=12" "QSB_TILE_PREFETCH=1 QSB_TILE_M=11" "QSB_TILE_PREFETCH=1 QSB_TILE_M=11 QSB_TILE_MINB=2" "QSB_TILE_PREFETCH=1 QSB_TILE_M=12 QSB_TILE_LOW=5" "QSB_TILE_PREFETCH=1 QSB_TILE_M=13"; do
  out=$(env $cfg timeout 300 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1)
  echo "$cfg :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["achieved"], d["roofline"]["frac"], d["config"]["passes"])' 2>&1)"
done
