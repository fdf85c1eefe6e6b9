cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_smoke7.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=1200 -rf > $O/r2_pytest_gpu7.log 2>&1; echo "pytest rc=$?" >> $O/r2_pytest_gpu7.log
for i in 1 2; do timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/r2_bench7_$i.log 2>&1; done
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --algo mma_sync --no-cpu-baseline > $O/r2_bench7_mma.log 2>&1
timeout 600 python scripts/big_n_ab.py > $O/r2_big_n_ab2.txt 2>&1
P="python bench.py --e2e-steps 0 --no-cpu-baseline --steps 3 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches7.csv $P > $O/r2_ncu7_l.log 2>&1
timeout 120 python scripts/profile_targets.py c3_tcgen05 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_tcgen05 -s 1 -c 1 -o $O/r2_prof_c3_tc05 -f python scripts/profile_targets.py c3_tcgen05 > $O/r2_ncu7_c3.log 2>&1
