#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rA -k "exact" > $O/pytest_exact.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_exact.log
B="timeout 120 python bench.py --e2e-steps 0 --no-cpu-baseline --steps 500 --warmup 30 --algo exact"
for a in "--exact-unroll 4 --exact-bps 4" "--exact-unroll 8 --exact-bps 3" "--exact-unroll 4 --exact-bps 8" "--exact-unroll 8 --exact-bps 6"; do
  $B $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', round(d['roofline']['achieved'],1), 'GB/s', round(d['ms_per_step']*1e3,1), 'us/step')"
done
