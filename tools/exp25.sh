timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense or pair or per_gate or final_state" 2>&1 | tail -3
timeout 600 python tools/kernel_probe.py --n 28 > gpurun_out/kp28b.jsonl 2> gpurun_out/kp28b.err; echo kp rc=$?
for p in dense unfused; do
  for e in "" "QSB_NO_PAIR256=1"; do
    env $e timeout 600 python bench.py --plan $p --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$p$e.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/b_$p$e.json')); print('$p', '$e', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['parity']['ok'])"
  done
done
