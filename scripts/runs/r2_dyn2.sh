# r02 §16: tests of the dynamic tail + the affected suites, then the fp8 A/B
set -x
timeout 1500 python -m pytest tests/test_gpu_tc05_dynamic.py tests/test_abi.py tests/test_gpu_parity.py tests/test_gpu_fp8.py tests/test_gpu_peer.py tests/test_gpu_pdl.py -x -q 2>&1 | tail -15
DTYPE=e4m3 DYNS="0 8" timeout 400 python scripts/tc05_dyn_ab.py 28 29 30 31 32 2>&1 | tee gpurun_out/tc05_dyn_ab_e4m3.txt
DYNS="0 8" timeout 400 python scripts/tc05_dyn_ab.py 24 27 28 30 33 2>&1 | tee gpurun_out/tc05_dyn_ab3.txt
