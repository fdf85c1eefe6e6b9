#!/bin/bash
# One ncu --set full capture per kernel family (each target first runs plain).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
declare -A K=( [c3_mma]=reduce_stream_kernel [c3_tcgen05]=reduce_tcgen05_kernel [c3_exact]=reduce_exact_kernel \
               [c5]=reduce_segmented_kernel [rows256]=reduce_rows_kernel [fp8_tcgen05]=reduce_tcgen05_kernel [bf16_mma]=reduce_stream_kernel )
for t in c3_mma c3_tcgen05 c3_exact c5 rows256 fp8_tcgen05 bf16_mma; do
  timeout 300 python scripts/profile_targets.py $t > $O/plain_$t.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K[$t]} -s 1 -c 1 -o $O/prof_$t -f \
      python scripts/profile_targets.py $t > $O/ncu_$t.log 2>&1
  echo "$t rc=$?"
done
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 3 --warmup 3"
$P > $O/plain_bench.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $P > $O/ncu_l.log 2>&1; echo "launches rc=$?"
