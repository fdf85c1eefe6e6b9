# Round-2 final evidence pass on the committed code (one gpurun call).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/fp6_smoke.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=1200 -rf > $O/fp6_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/fp6_pytest_gpu.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/fp6_bench.log 2>&1
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/fp6_bench_ref.log 2>&1
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 > $O/fp6_bench_c5.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --dtype e4m3 > $O/fp6_bench_e4m3.log 2>&1
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 3 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fp6_launches_default.csv $P > $O/fp6_ncu_l.log 2>&1
timeout 120 python scripts/profile_targets.py rows256 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_rows_tc05 -s 1 -c 1 -o $O/fp6_prof_rows256 -f python scripts/profile_targets.py rows256 > $O/fp6_ncu_rows.log 2>&1
tail -3 $O/fp6_pytest_gpu.log; tail -1 $O/fp6_smoke.log; cut -c1-300 $O/fp6_bench.log | tail -1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --algo exact > $O/fp6_bench_exact.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --algo exact --dtype e4m3 > $O/fp6_bench_exact_e4m3.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --dtype bf16 > $O/fp6_bench_bf16.log 2>&1
