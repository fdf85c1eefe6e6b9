for v in none spin copy e2e self none spin; do python scripts/warm_fresh.py $v; done
for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('20/5 e2e-first', d['ms_per_step'], d['clocks'], d['e2e'])"; done
