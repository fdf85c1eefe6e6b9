set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
lscpu | head -20; free -g
for i in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('20/5', d['ms_per_step'], d['clocks'])"; done
for i in 1 2; do python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('1000/20', d['ms_per_step'], d['clocks'])"; done
for i in 1 2; do python bench.py --steps 20 --warmup 200 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('20/200', d['ms_per_step'], d['clocks'])"; done
