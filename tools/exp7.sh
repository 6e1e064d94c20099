export QSB_BENCH_PASSES=1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pp_choose.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/pp_choose.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['frac'], d['parity']['ok'], r['launch_ms'])"
python -m pytest tests/test_bench_parity.py -x -q 2>&1 | tail -3
python bench.py --workload random28 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('random28', d['value'], d['parity'])"
