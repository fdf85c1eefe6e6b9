#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16.py tests/test_gpu_fp8.py -m gpu -q -x -k "bulk or config_knobs or full_size_c3" > $O/pytest_bulk.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_bulk.log
B="timeout 120 python bench.py --e2e-steps 0 --no-cpu-baseline --steps 500 --warmup 30"
for a in "--algo mma_sync" "--algo bulk" "--algo bulk --bulk-stages 12 --bulk-ctas 1" "--algo bulk --bulk-stages 4 --bulk-kb 24 --bulk-ctas 2" "--algo bulk --bulk-stages 8 --bulk-kb 8 --bulk-ctas 2" "--algo bulk --bulk-stages 3 --bulk-kb 32 --bulk-ctas 2" "--algo bulk --bulk-stages 4 --bulk-kb 16 --bulk-ctas 3" "--algo bulk --dtype e4m3" "--algo tcgen05 --dtype e4m3"; do
  $B $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', round(d['roofline']['achieved'],1), 'GB/s', round(d['ms_per_step']*1e3,1), 'us/step')"
done
