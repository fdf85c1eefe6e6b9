cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out
B="python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline"
for i in 1 2 3 4; do
  for a in default mma_sync; do
    echo "$a $(timeout 300 $B --algo $a 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["algo"], round(d["ms_per_step"]*1e3,2), round(d["roofline"]["achieved"],1), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
  done
done > $O/r2_default_ab.txt 2>&1
