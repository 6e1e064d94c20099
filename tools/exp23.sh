for g in 1 2 3; do
  python bench.py --local-shards $g --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ls$g.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ls$g.json')); r=d['roofline']; print($g, d['value'], d['ms_per_step'], d['config']['passes'], r.get('exchanges_per_step'), r.get('exchange_ms_total'), d['parity']['ok'])"
done
