export QSB_JIT_DEBUG=1 QSB_JIT_CACHE=/tmp/jc5
rm -rf /tmp/jc5
python -c "
import bench
print(bench.e2e_cold('qft30', 0, '/tmp/jc5', 495))
" 2>&1 | tail -3
ls /tmp/jc5 | wc -l
python - <<'PY'
import subprocess, sys, bench, os
env = dict(os.environ)
r = subprocess.run([sys.executable, "-c", bench.COLD_PROBE % {"root": bench.ROOT, "workload": "qft30", "device": 0}], capture_output=True, text=True, env=env)
print(r.stdout[-500:]); print(r.stderr[-3000:])
PY
