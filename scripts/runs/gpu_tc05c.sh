#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
B="timeout 120 python bench.py --e2e-steps 0 --no-cpu-baseline --steps 500 --warmup 30"
for a in "--algo mma_sync --unroll 8 --bps 8" "--algo mma_sync --unroll 8 --bps 4" "--algo mma_sync --unroll 4 --bps 8" \
         "--algo tcgen05 --stages 4 --stage-kb 16 --slots 4 --ctas 3" "--algo tcgen05 --stages 4 --stage-kb 16 --slots 2 --ctas 3" \
         "--algo tcgen05 --stages 3 --stage-kb 20 --slots 4 --ctas 3" "--algo tcgen05 --stages 5 --stage-kb 12 --slots 4 --ctas 3" \
         "--algo tcgen05 --stages 6 --stage-kb 8 --slots 4 --ctas 3" "--algo tcgen05 --stages 3 --stage-kb 16 --slots 4 --ctas 3" \
         "--algo tcgen05 --stages 2 --stage-kb 32 --slots 4 --ctas 3" "--algo tcgen05 --stages 4 --stage-kb 16 --slots 4 --ctas 3 --tc-chain 2" \
         "--algo tcgen05 --stages 4 --stage-kb 16 --slots 4 --ctas 3 --prefetch 2" "--algo tcgen05 --stages 8 --stage-kb 8 --slots 4 --ctas 3" \
         "--algo tcgen05 --stages 3 --stage-kb 12 --slots 4 --ctas 4" "--algo tcgen05 --stages 2 --stage-kb 20 --slots 4 --ctas 4" \
         "--algo shuffle --unroll 16 --bps 4" "--algo mma_sync --unroll 8 --bps 8" "--algo tcgen05 --stages 4 --stage-kb 16 --slots 4 --ctas 3"; do
  $B $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', round(d['roofline']['achieved'],1), 'GB/s', round(d['ms_per_step']*1e3,1), 'us/step', d['clocks']['sm_mhz'])"
done 2>&1 | tee gpurun_out/tc05_sweep2.txt
