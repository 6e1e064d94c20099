for e in "" "QSB_EXP_OOP_ALL=1" "" "QSB_EXP_OOP_ALL=1"; do
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sr.json 2>gpurun_out/sr.err
  python -c "import json; d=json.load(open('gpurun_out/sr.json')); print('$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'], d['config']['passes'])" || tail -3 gpurun_out/sr.err
done
QSB_EXP_OOP_ALL=1 python tools/pass_profile.py --n 30 > gpurun_out/pass_profile_oop.jsonl 2>gpurun_out/pp.err
python tools/pass_profile.py --n 30 > gpurun_out/pass_profile_inplace.jsonl 2>/dev/null
