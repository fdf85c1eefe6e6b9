#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 120 ./scripts/tc05_issue 2>&1 | tee gpurun_out/tc05_issue.txt
B="timeout 120 python bench.py --algo tcgen05 --e2e-steps 0 --no-cpu-baseline --steps 300 --warmup 20"
for a in "--stages 6 --stage-kb 16 --slots 8 --ctas 2" "--stages 4 --stage-kb 24 --slots 8 --ctas 2" "--stages 3 --stage-kb 32 --slots 8 --ctas 2" \
         "--stages 4 --stage-kb 16 --slots 4 --ctas 3" "--stages 3 --stage-kb 16 --slots 4 --ctas 4" "--stages 6 --stage-kb 8 --slots 4 --ctas 4" \
         "--stages 4 --stage-kb 12 --slots 4 --ctas 4" "--stages 2 --stage-kb 24 --slots 4 --ctas 4" "--stages 3 --stage-kb 16 --slots 4 --ctas 4 --tc-chain 8"; do
  $B $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', round(d['roofline']['achieved'],1), 'GB/s')"
done 2>&1 | tee gpurun_out/tc05_ctas.txt
