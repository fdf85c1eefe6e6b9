cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_smoke2.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=1200 -rf > $O/r2_pytest_gpu_full2.log 2>&1; echo "pytest rc=$?" >> $O/r2_pytest_gpu_full2.log
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 --warmup 5"
( timeout 300 $B; timeout 300 $B --algo tcgen05; timeout 300 $B --algo exact; timeout 300 $B --algo exact --dtype bf16; timeout 300 $B --dtype e4m3 ) > $O/r2_bench_set.log 2>&1
timeout 600 python scripts/c2_compare.py > $O/r2_c2_compare2.log 2>&1
