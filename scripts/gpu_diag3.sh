python -c "import __graft_entry__ as g; g.build()" > /dev/null
for d in full none; do echo "== deps $d"; HM_DIAG_DEPS=$d HM_ENGINE_STATS=1 timeout 300 python scripts/engine_stats.py 2>&1 | grep -A12 "engine stats" | grep -v "^---" | awk '/engine stats/{n++} n%3==0' ; done
