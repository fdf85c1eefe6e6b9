cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_fp8.py tests/test_gpu_bf16.py tests/test_gpu_pdl.py tests/test_gpu_precision.py -q -p no:cacheprovider -x > $O/r2_pytest_pre.log 2>&1; echo rc=$? >> $O/r2_pytest_pre.log
timeout 600 python scripts/tc05_vs_mma_ab.py > $O/r2_tc05_vs_mma3.txt 2>&1
timeout 300 python scripts/tc05_small_sweep_r2.py > $O/r2_tc05_small2.txt 2>&1
for a in tcgen05 mma_sync tcgen05 mma_sync; do timeout 120 python scripts/warm_fresh.py none $a; done > $O/r2_warm_algos2.txt 2>&1
