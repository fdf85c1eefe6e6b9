#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for cfg in "8 16 16 4 1" "8 16 1 4 1" "4 32 16 4 1" "3 64 16 4 1" "12 16 16 4 1" "6 16 8 4 2"; do
  timeout 60 ./scripts/tc05_trace $cfg
done 2>&1 | tee gpurun_out/tc05_trace.txt
B="timeout 120 python bench.py --algo tcgen05 --e2e-steps 0 --no-cpu-baseline --steps 300 --warmup 20"
for a in "--stages 8 --stage-kb 16" "--stages 4 --stage-kb 32" "--stages 3 --stage-kb 64" "--stages 6 --stage-kb 16 --slots 8 --ctas 2"; do
  $B $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', round(d['roofline']['achieved'],1), 'GB/s')"
done 2>&1 | tee -a gpurun_out/tc05_trace.txt
