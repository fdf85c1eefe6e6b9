# r02 §16: the rewritten dynamic-tail completion (thread 0 CTA sum + ticket, last CTA loads all partials at once)
export TRACE_REPS=200
for d in 0 8; do TRACE_DYN=$d timeout 60 scripts/tc05_trace 4 32 4 2 1 30 | grep -E "^cfg|^CTAs|deciles|completion"; done
timeout 900 python -m pytest tests/test_gpu_tc05_dynamic.py tests/test_gpu_peer.py -x -q 2>&1 | tail -3
DYNS="8" timeout 400 python scripts/tc05_dyn_ab.py 27 28 30 32 2>&1 | tee gpurun_out/tc05_dyn_ab4.txt
