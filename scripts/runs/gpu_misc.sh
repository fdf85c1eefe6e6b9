#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; O=gpurun_out
timeout 300 python -m pytest tests/test_capi.py -m gpu -q > $O/pytest_capi.log 2>&1; echo "capi rc=$?"; tail -1 $O/pytest_capi.log
timeout 600 python scripts/c2_sweep.py 2>&1 | tee $O/c2_sweep.txt
