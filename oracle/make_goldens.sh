#!/usr/bin/env bash
# Regenerates tests/golden/ from the unmodified reference (needs /root/reference).
# 1. builds the reference's headers + our eigen_lite / mini_gtest shims into oracle/_ref
# 2. runs the reference's own GoogleTest suites against that build (shim check)
# 3. emits the golden vectors through the reference's public API.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
make -C "$ROOT/oracle" -j8 ref oracle
for t in smoke core statevector simulator noise pathsum transpile mapping ir variational bench; do
  "$ROOT/oracle/_ref/${t}_test" > /dev/null
done
mkdir -p "$ROOT/tests/golden"
"$ROOT/oracle/_ref/ref_driver" golden "$ROOT/tests/golden"
"$ROOT/oracle/_ref/ref_driver" golden_big "$ROOT/tests/golden"
# Full-size benchmarked configurations (random28, qft30, random30): ~20 min on
# 8 cores and ~32 GiB of host RAM, so only with GOLDEN_HUGE=1.
if [ "${GOLDEN_HUGE:-0}" = 1 ]; then
  mkdir -p "$ROOT/tests/golden/huge"
  "$ROOT/oracle/_ref/ref_driver" golden_huge "$ROOT/tests/golden/huge" random28 qft30 random30
fi
"$ROOT/oracle/_ref/ref_driver" golden_cut "$ROOT/tests/golden"
