cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_smoke3.log 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 50 --warmup 10 --algo exact"
for u in 4 8; do for b in 2 3 4 5; do
  echo "unroll=$u bps=$b $(timeout 300 $B --exact-unroll $u --exact-bps $b 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["achieved"],1), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done; done > $O/r2_exact_sweep.txt 2>&1
