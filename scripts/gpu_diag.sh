# C2 engine diagnostics: build, per-pass trace, per-role stats, program shapes
python -c "import __graft_entry__ as g; g.build()" > /dev/null
CUT=0 timeout 200 python scripts/trace_step.py 2>&1 | tail -10
HM_ENGINE_STATS=1 timeout 300 python scripts/engine_stats.py 2>&1 | grep "engine stats" | awk 'NR%3==0'
HM_ENGINE_STATS=2 timeout 300 python scripts/engine_stats.py 2>&1 | grep -v "^---" | sort | uniq | head -40
