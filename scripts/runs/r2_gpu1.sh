python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=1200 -rf > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
python scripts/c2_compare.py > gpurun_out/r2_c2_compare.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1
