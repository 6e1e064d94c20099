# the reference CPU simulator on this host, configs 1, 2, 5
# (all threads; config 1 also with 1 thread), then the same configs on the GPU.
set -x
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" > gpurun_out/cpu_host.txt; nproc >> gpurun_out/cpu_host.txt
for c in config1 config5 config2; do
  ./oracle/_ref/ref_driver bench_config $c >> gpurun_out/cpu_configs.jsonl
done
OMP_NUM_THREADS=1 ./oracle/_ref/ref_driver bench_config config1 >> gpurun_out/cpu_configs.jsonl
python tools/config_sweep.py > gpurun_out/gpu_configs.jsonl 2> gpurun_out/gpu_configs.err
cat gpurun_out/cpu_host.txt gpurun_out/cpu_configs.jsonl gpurun_out/gpu_configs.jsonl; tail -3 gpurun_out/gpu_configs.err
