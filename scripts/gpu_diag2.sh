python -c "import __graft_entry__ as g; g.build()" > /dev/null
for d in full none intra cross; do echo "== deps $d"; HM_DIAG_DEPS=$d CUT=0 timeout 200 python scripts/trace_step.py 2>&1 | tail -8; done
