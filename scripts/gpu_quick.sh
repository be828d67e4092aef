# quick perf iteration: build, C2 parity subset, per-pass trace, short bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "config2 or solve_and_flux or repeat" 2>&1 | tail -3
CUT=0 timeout 200 python scripts/trace_step.py 2>&1 | tail -8
timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-level-form 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bench', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['config']['engine_ms'], d['e2e']['value'])"

