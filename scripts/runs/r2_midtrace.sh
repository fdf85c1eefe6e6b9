export TRACE_REPS=200
for lg in 24 26 27 28; do timeout 60 scripts/stream_trace $lg 8; done
for lg in 26 27 28; do for d in 0 8; do TRACE_DYN=$d timeout 60 scripts/tc05_trace 4 32 4 2 1 $lg | grep -E "^cfg|^CTAs|deciles"; done; done
