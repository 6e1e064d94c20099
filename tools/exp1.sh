set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
./build/l2_probe > gpurun_out/l2_probe.jsonl 2>&1
python tools/pass_sizes.py 20 21 22 23 24 26 > gpurun_out/pass_sizes_auto.jsonl 2>&1
QSB_TILE_M=13 python tools/pass_sizes.py 20 21 22 23 24 > gpurun_out/pass_sizes_m13.jsonl 2>&1
QSB_TILE_LOW=3 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_low3.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_low4.json 2>&1
cat gpurun_out/*.jsonl gpurun_out/bench_low*.json
