#!/bin/bash
# Full GPU pass: smoke, all -m gpu tests, bench (default + per algo), C2
# comparison, c5 bench, ncu launch list + one --set full capture per kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out; O=gpurun_out
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
echo "== pytest"; timeout 2400 python -m pytest tests -m gpu -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
echo "== bench default"; timeout 300 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"; cat $O/bench.log
for a in mma_sync tcgen05 shuffle; do timeout 300 python bench.py --algo $a --e2e-steps 0 --no-cpu-baseline --steps 500 --warmup 30 > $O/bench_$a.log 2>&1; done
echo "== bench c5"; timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; echo "c5 rc=$?"
echo "== ref arm"; timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.log 2>&1; echo "ref rc=$?"
echo "== c2"; timeout 300 python scripts/c2_compare.py > $O/c2_compare.txt 2>&1; cat $O/c2_compare.txt
echo "== ncu"
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 3 --warmup 2"
$P > $O/plain.log 2>&1 && $P --algo tcgen05 > $O/plain_t.log 2>&1 && $P --workload c5 > $O/plain_c5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $P > $O/ncu_l.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_stream_kernel -s 2 -c 1 -o $O/prof_mma_sync -f $P > $O/ncu_m.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_tcgen05_kernel -s 2 -c 1 -o $O/prof_tcgen05 -f $P --algo tcgen05 > $O/ncu_t.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reduce_segmented_kernel -s 2 -c 1 -o $O/prof_c5 -f $P --workload c5 > $O/ncu_c5.log 2>&1
echo "ncu rc=$?"
