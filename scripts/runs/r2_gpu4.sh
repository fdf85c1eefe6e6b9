cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_segmented_batches.py tests/test_gpu_segmented.py tests/test_gpu_fp8.py -q -p no:cacheprovider -k "batched or rows" > $O/r2_pytest_rows.log 2>&1; echo "pytest rc=$?" >> $O/r2_pytest_rows.log
timeout 600 python scripts/batched_b2b.py > $O/r2_batched_b2b.txt 2>&1
timeout 900 python scripts/speedup_curve.py > $O/r2_speedup_curve.log 2>&1
