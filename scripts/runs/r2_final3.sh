# Round-2 final evidence pass after the default went back to mma.sync (one gpurun call).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/final3_smoke.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=1200 -rf > $O/final3_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/final3_pytest_gpu.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/final3_bench.log 2>&1
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/final3_bench_ref.log 2>&1
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 > $O/final3_bench_c5.log 2>&1
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 3 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/final3_launches_default.csv $P > $O/final3_ncu_l.log 2>&1
timeout 120 python scripts/profile_targets.py c3_mma > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_stream_kernel -s 1 -c 1 -o $O/final3_prof_c3_mma -f python scripts/profile_targets.py c3_mma > $O/final3_ncu_c3.log 2>&1
