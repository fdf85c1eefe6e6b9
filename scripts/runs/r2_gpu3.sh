cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
timeout 60 ./scripts/tc05_borient > $O/r2_tc05_borient.txt 2>&1; echo "borient rc=$?" >> $O/r2_tc05_borient.txt
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 --warmup 5"
( timeout 300 $B --algo exact; timeout 300 $B --algo exact --dtype bf16; timeout 300 $B --algo exact --dtype e4m3; timeout 300 $B --algo mma_sync --dtype e4m3 ) > $O/r2_bench_exact.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_exact.py tests/test_gpu_bf16.py tests/test_gpu_fp8.py tests/test_gpu_segmented.py tests/test_gpu_segmented_batches.py tests/test_gpu_peer.py -q -p no:cacheprovider -x > $O/r2_pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> $O/r2_pytest_gpu3.log
for t in c2_mma c2_shuffle c2_tcgen05; do
  timeout 120 python scripts/profile_targets.py $t > /dev/null 2>&1 && \
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum \
     --clock-control none --cache-control all -k regex:reduce_ --csv python scripts/profile_targets.py $t > $O/r2_ncu_$t.csv 2>&1
done
timeout 120 python scripts/profile_targets.py c3_mma > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_stream_kernel -s 1 -c 1 -o $O/r2_prof_c3_mma -f python scripts/profile_targets.py c3_mma > $O/r2_ncu_c3_mma.log 2>&1
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 3 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches_default.csv $P > $O/r2_ncu_l.log 2>&1
