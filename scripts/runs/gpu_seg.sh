#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "segmented or batched or edge or loguniform or index or bf16_segmented" > $O/pytest_seg.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_seg.log
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; python -c "import json; d=json.load(open('$O/bench_c5.log')); print('c5', d['roofline']['achieved'], d['roofline']['kernel_ms'])"
timeout 500 python scripts/batched_bench.py 2>&1 | tee $O/batched_bench.txt
