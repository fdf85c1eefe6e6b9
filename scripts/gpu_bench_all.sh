#!/bin/bash
# Every bench line of DESIGN §9 on one box, then the default command's ncu launch list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "default rc=$?"
for a in "mma_sync" "tcgen05" "shuffle" "bulk" "exact"; do
  timeout 300 python bench.py --algo $a --no-cpu-baseline --e2e-steps 0 > $O/bench_$a.log 2>&1; echo "$a rc=$?"
done
timeout 300 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.log 2>&1; echo "c5 rc=$?"
timeout 300 python bench.py --dtype bf16 --no-cpu-baseline > $O/bench_bf16.log 2>&1; echo "bf16 rc=$?"
timeout 300 python bench.py --dtype e4m3 --no-cpu-baseline > $O/bench_e4m3.log 2>&1; echo "e4m3 rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_arm.log 2>&1; echo "reference rc=$?"
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 3 --warmup 3"
$P > $O/plain_bench.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $P > $O/ncu_l.log 2>&1; echo "launches rc=$?"
