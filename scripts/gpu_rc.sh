python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "recompress or multi_rhs" 2>&1 | tail -4
timeout 300 python scripts/mrhs_bench.py 2>&1 | tail -3
timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); c=d['config']; print('bench', d['value'], d['ms_per_step'], d['roofline']['achieved'], c['engine_ms']); print('recompressed', c['recompressed']); print('level', c['level_form'])"
