#!/bin/bash
# First-contact GPU check: smoke, parity tests (tcgen05 isolated), benches,
# ncu launch list.  Every step under its own timeout; logs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi > $O/nvidia_smi.txt 2>&1
nproc > $O/host_nproc.txt; lscpu > $O/host_lscpu.txt 2>&1
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
echo "== pytest (no tcgen05)"; timeout 1500 python -m pytest tests -m gpu -q -rA -k "not tcgen05 and not full_size_c3 and not config_knobs" > $O/pytest_gpu_a.log 2>&1; echo "pytest_a rc=$?"
echo "== pytest (tcgen05)"; timeout 600 python -m pytest tests -m gpu -q -rA -k "tcgen05" > $O/pytest_gpu_tc.log 2>&1; echo "pytest_tc rc=$?"
echo "== pytest (full size / knobs)"; timeout 900 python -m pytest tests -m gpu -q -rA -k "full_size_c3 or config_knobs" > $O/pytest_gpu_b.log 2>&1; echo "pytest_b rc=$?"
for a in mma_sync shuffle tcgen05; do
  echo "== bench $a"; timeout 300 python bench.py --algo $a --steps 200 --warmup 10 > $O/bench_$a.log 2>&1; echo "bench $a rc=$?"
done
echo "== bench c5"; timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; echo "bench c5 rc=$?"
echo "== ncu launches"
timeout 300 python bench.py --algo mma_sync --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --algo mma_sync --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/ncu.log 2>&1
echo "ncu rc=$?"
tail -n 3 $O/*.log
