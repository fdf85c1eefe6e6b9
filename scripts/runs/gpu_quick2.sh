#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rA -k "segmented or batched or edge or loguniform or index or config_knobs" > $O/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_q.log
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; python -c "import json; d=json.load(open('$O/bench_c5.log')); print('c5', d['roofline']['achieved'], d['roofline']['kernel_ms'])"
B="timeout 120 python bench.py --e2e-steps 0 --no-cpu-baseline --steps 500 --warmup 30"
for a in "--algo tcgen05" "--algo tcgen05 --interleave 1" "--algo tcgen05 --interleave 1 --stages 3 --stage-kb 20" "--algo mma_sync"; do
  $B $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', round(d['roofline']['achieved'],1), 'GB/s', round(d['ms_per_step']*1e3,1), 'us/step')"
done
