#!/bin/bash
# Full -m gpu suite + smoke + the driver's bench command on the committed code.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1
tail -2 gpurun_out/pytest_gpu_full.log; tail -1 gpurun_out/smoke.log; tail -1 gpurun_out/bench_default.log
