cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=1200 -rf > $O/r2_pytest_gpu6.log 2>&1; echo "pytest rc=$?" >> $O/r2_pytest_gpu6.log
timeout 800 python scripts/tc05_vs_mma_ab.py > $O/r2_tc05_vs_mma2.txt 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 --warmup 5"
( timeout 300 $B --algo tcgen05; timeout 300 $B --algo tcgen05 --dtype bf16; timeout 300 $B --algo tcgen05 --dtype e4m3; timeout 300 $B ) > $O/r2_bench_tc05.log 2>&1
timeout 900 python scripts/speedup_curve.py > $O/r2_speedup_curve2.log 2>&1
