python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for t in 1 2 4 8; do
  echo "== tdiv $t"; HM_PIECE_TDIV=$t CUT=0 timeout 200 python scripts/trace_step.py 2>&1 | tail -3
  HM_PIECE_TDIV=$t timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-level-form 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bench', d['value'], d['ms_per_step'], d['config']['engine_ms'])"
done
