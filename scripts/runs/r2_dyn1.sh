export TRACE_REPS=200
for d in 0 10 25 50 100; do TRACE_DYN=$d timeout 60 scripts/tc05_trace 4 32 4 2 1 30 | grep -E "^cfg|^CTAs|deciles|completion"; done
TRACE_DYN=25 TRACE_REPS=30 timeout 60 scripts/tc05_trace 4 32 4 2 1 33 | grep -E "^cfg|^CTAs|deciles"
timeout 900 python -m pytest tests/test_gpu_tc05_dynamic.py -x -q 2>&1 | tail -15
