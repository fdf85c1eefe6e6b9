#!/bin/bash
# tcgen05 variants: correctness first (pytest -k tcgen05), then the sweep.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out; O=gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rA -k "tcgen05 or config_knobs" > $O/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_tc.log
B="timeout 120 python bench.py --algo tcgen05 --e2e-steps 0 --no-cpu-baseline --steps 300 --warmup 20"
: > $O/sweep_tc.jsonl
while read -r args; do
  $B $args >> $O/sweep_tc.jsonl 2>>$O/sweep_tc.err || echo "FAIL $args" >> $O/sweep_tc.err
done <<'CFG'
--stages 8 --stage-kb 16 --slots 1 --tc-chain 4
--stages 8 --stage-kb 16 --slots 16 --tc-chain 4
--stages 8 --stage-kb 16 --slots 16 --tc-chain 4 --split 4
--stages 8 --stage-kb 16 --slots 16 --tc-chain 4 --prefetch 8
--stages 8 --stage-kb 16 --slots 16 --tc-chain 4 --prefetch 16
--stages 6 --stage-kb 16 --slots 8 --tc-chain 4 --ctas 2
--stages 4 --stage-kb 32 --slots 8 --tc-chain 4 --ctas 2
--stages 6 --stage-kb 32 --slots 16 --tc-chain 4
--stages 3 --stage-kb 64 --slots 16 --tc-chain 4
--stages 3 --stage-kb 64 --slots 16 --tc-chain 4 --split 8
--stages 3 --stage-kb 64 --slots 16 --tc-chain 4 --prefetch 4
--stages 12 --stage-kb 16 --slots 16 --tc-chain 4 --prefetch 8
--stages 24 --stage-kb 8 --slots 16 --tc-chain 4 --prefetch 16
--stages 6 --stage-kb 32 --slots 16 --tc-chain 4 --prefetch 8
CFG
python - <<'PY'
import json
for l in open("gpurun_out/sweep_tc.jsonl"):
    try: d = json.loads(l)
    except Exception: continue
    k = d["config"]["knobs"]
    print(f'{k["tc05_stages"]:2d}x{k["tc05_stage_kb"]:2d}KB slots={k["tc05_slots"]:2d} chain={k["tc05_chain"]} ctas={k["tc05_ctas"]} pf={k["tc05_prefetch"]:2d} split={k["tc05_split"]}  '
          f'kernel {d["roofline"]["achieved"]:7.1f} GB/s  {d["value"]:7.1f} Gelem/s  clk {d["clocks"]["sm_mhz"]}')
PY
cat $O/sweep_tc.err | tail -5
