python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for cfg in "2 4" "1 4" "1 8" "2 8" "1 16"; do set -- $cfg
  echo "== div $1 min $2"; HM_PIECE_DIV=$1 HM_PIECE_MIN=$2 CUT=0 timeout 200 python scripts/trace_step.py 2>&1 | tail -7
  HM_PIECE_DIV=$1 HM_PIECE_MIN=$2 timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-level-form 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bench', d['value'], d['ms_per_step'], d['config']['engine_ms'])"
done
