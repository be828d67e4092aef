python -c "import __graft_entry__ as g; g.build()" > /dev/null
for d in full none intra cross; do echo "== deps $d"; HM_DIAG_DEPS=$d timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --no-level-form 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bench', d['ms_per_step'], d['config']['engine_ms'])"; done
