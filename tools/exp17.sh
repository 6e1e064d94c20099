export QSB_TMA=1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiled or knob or fused or basis or from_basis" 2>&1 | tail -5
timeout 300 python -m pytest tests/test_bench_parity.py -x -q -k "random28 or qft30" 2>&1 | tail -3
unset QSB_TMA
export QSB_BENCH_PASSES=1
for v in "QSB_TMA=0" "QSB_TMA=1" "QSB_TMA=0" "QSB_TMA=1"; do
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tma_${v}.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/tma_${v}.json')); r=d['roofline']
print('$v', d['value'], d['ms_per_step'], r['frac'], d['clocks']['sm_mhz'], d['parity']['ok'], r['launch_ms'])" | cut -c1-400
done
