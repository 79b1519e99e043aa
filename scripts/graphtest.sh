python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for a in "" "--graph"; do python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $a 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$a', round(d['ms_per_step'],4), d['cuda_graph'])"; done
