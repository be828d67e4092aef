python -c "import __graft_entry__ as g; g.build()"
HM_ENGINE_STATS=1 timeout 300 python scripts/engine_stats.py 2>&1 | grep -A1 "^---" | grep engine | awk 'NR%3==0'
