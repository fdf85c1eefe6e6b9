#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rA -k "exact or c4_on_one_gpu" > $O/pytest_exact.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_exact.log
B="timeout 120 python bench.py --e2e-steps 0 --no-cpu-baseline --steps 500 --warmup 30"
for a in "--algo exact" "--algo mma_sync"; do
  $B $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', round(d['roofline']['achieved'],1), 'GB/s', round(d['ms_per_step']*1e3,1), 'us/step', d['result'])"
done
echo "== memcheck"
timeout 300 python scripts/sanitize_smoke.py > $O/sanitize_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --leak-check no python scripts/sanitize_smoke.py > $O/memcheck.log 2>&1
echo "memcheck rc=$?"; tail -5 $O/memcheck.log
