cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 50 --warmup 10"
for lg in 24 26 28 30 31; do for a in mma_sync tcgen05; do for d in e4m3 e5m2; do
  echo "n=2^$lg $d $a $(timeout 300 $B --dtype $d --algo $a --n-total $((1<<lg)) 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2), "us", round(d["roofline"]["achieved"],1), "GB/s", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done; done; done > $O/r2_fp8_default.txt 2>&1
