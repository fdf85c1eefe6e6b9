#!/bin/bash
# Tuning sweep + read ceiling + one ncu --set full capture per kernel family.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out; O=gpurun_out
B="timeout 120 python bench.py --e2e-steps 0 --no-cpu-baseline --steps 300 --warmup 20"
echo "== read ceiling"; timeout 120 ./scripts/read_ceiling > $O/read_ceiling.txt 2>&1; cat $O/read_ceiling.txt
echo "== torch.sum"; timeout 120 python scripts/torch_sum_baseline.py > $O/torch_sum.txt 2>&1; cat $O/torch_sum.txt
: > $O/sweep.jsonl
for u in 4 8 16; do for b in 2 4 8; do for c in 1 4; do
  $B --algo mma_sync --unroll $u --bps $b --chain $c >> $O/sweep.jsonl 2>>$O/sweep.err
done; done; done
for u in 8 16; do for b in 4 8; do $B --algo shuffle --unroll $u --bps $b >> $O/sweep.jsonl 2>>$O/sweep.err; done; done
for sk in "8 16" "12 16" "13 16" "6 32" "4 48" "3 64" "24 8" "16 8" "10 20" "7 32" "5 40"; do
  set -- $sk; $B --algo tcgen05 --stages $1 --stage-kb $2 >> $O/sweep.jsonl 2>>$O/sweep.err
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep.jsonl"):
    try: d = json.loads(l)
    except Exception: continue
    k = d["config"]["knobs"]
    print(f'{d["config"]["algo"]:9s} u={k["unroll"]:2d} bps={k["blocks_per_sm"]} chain={k["chain"]} st={k["tc05_stages"]:2d}x{k["tc05_stage_kb"]:2d}KB  '
          f'kernel {d["roofline"]["achieved"]:7.1f} GB/s  step {d["ms_per_step"]*1e3:6.1f} us  {d["value"]:7.1f} Gelem/s  clk {d["clocks"]["sm_mhz"]}')
PY
echo "== ncu full (mma_sync, tcgen05)"
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 2 --warmup 1"
$P --algo mma_sync > $O/plain_m.log 2>&1 && $P --algo tcgen05 > $O/plain_t.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_stream_kernel -s 1 -c 1 -o $O/prof_mma_sync -f $P --algo mma_sync > $O/ncu_m.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_tcgen05_kernel -s 1 -c 1 -o $O/prof_tcgen05 -f $P --algo tcgen05 > $O/ncu_t.log 2>&1
echo "ncu rc=$?"
