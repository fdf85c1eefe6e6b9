#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rA -k "segmented or config_knobs or precision or batched or edge or loguniform or index" > $O/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_q.log
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; python -c "import json; d=json.load(open('$O/bench_c5.log')); print('c5', d['roofline']['achieved'], d['roofline']['kernel_ms'])"
timeout 300 python scripts/c2_compare.py 2>&1 | tee $O/c2_compare.txt
