# r02 §16 evidence pass with the tcgen05 dynamic tail as the large-n default (one gpurun call).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/dyn_smoke.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/dyn_bench.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --algo mma_sync > $O/dyn_bench_mma.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/dyn_bench2.log 2>&1
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 3 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dyn_launches_default.csv $P > $O/dyn_ncu_l.log 2>&1
timeout 120 python scripts/profile_targets.py c3_tcgen05 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_tcgen05_kernel -s 1 -c 1 -o $O/dyn_prof_c3_tcgen05 -f python scripts/profile_targets.py c3_tcgen05 > $O/dyn_ncu_c3.log 2>&1
timeout 120 python scripts/profile_targets.py fp8_tcgen05 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_tcgen05_kernel -s 1 -c 1 -o $O/dyn_prof_fp8_tcgen05 -f python scripts/profile_targets.py fp8_tcgen05 > $O/dyn_ncu_fp8.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=1200 -rf > $O/dyn_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/dyn_pytest_gpu.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/dyn_bench_ref.log 2>&1
tail -3 $O/dyn_pytest_gpu.log; tail -1 $O/dyn_smoke.log; cut -c1-400 $O/dyn_bench.log | tail -2
