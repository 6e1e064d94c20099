# register-width cost: new (0.99) vs old (1.05) on random28 / random30, alternating in one call
for w in random28 random30; do
for e in "" "QSB_PASS_COST_R5=1.05" "" "QSB_PASS_COST_R5=1.05"; do
  env $e timeout 600 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$w', '$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'])" || tail -3 gpurun_out/sr.err
done
done
