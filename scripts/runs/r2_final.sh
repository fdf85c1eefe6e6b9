# Round-2 final evidence pass (one gpurun call): smoke, all -m gpu tests, the
# driver's bench command (ours + reference arm), the ncu launch list and one
# ncu --set full capture of the default kernel, C2 compare.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=1200 -rf > $O/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/final_pytest_gpu.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/final_bench.log 2>&1
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/final_bench_ref.log 2>&1
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 > $O/final_bench_c5.log 2>&1
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 3 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/final_launches_default.csv $P > $O/final_ncu_l.log 2>&1
timeout 120 python scripts/profile_targets.py c3_mma > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_stream_kernel -s 1 -c 1 -o $O/final_prof_c3_mma -f python scripts/profile_targets.py c3_mma > $O/final_ncu_c3.log 2>&1
timeout 120 python scripts/profile_targets.py rows256 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:reduce_row -s 1 -c 1 -o $O/final_prof_rows256 -f python scripts/profile_targets.py rows256 > $O/final_ncu_rows.log 2>&1
