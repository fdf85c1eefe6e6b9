#!/bin/bash
# Full check: smoke, every -m gpu test, default bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
python -c "import __graft_entry__ as g; g.build_c_demo()" > /dev/null 2>&1
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
echo "== pytest"; timeout 2400 python -m pytest tests -m gpu -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|ERROR" $O/pytest_gpu.log | head; tail -1 $O/pytest_gpu.log
echo "== bench"; timeout 300 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"; cat $O/bench.log
