# piece sizing with the 3-stage engine (env knobs, no rebuild): C2 flux
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for cfg in "2 4" "1 4" "4 4" "2 2" "2 8"; do
  set -- $cfg
  echo "== HM_PIECE_DIV=$1 HM_PIECE_MIN=$2"
  for r in 1 2; do
    HM_PIECE_DIV=$1 HM_PIECE_MIN=$2 timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --no-level-form 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('flux us', round(d['ms_per_step']*1e3,1), 'engine us', round(d['config']['engine_ms']['flux']*1e3,1), 'units', d['config']['engine']['units'])"
  done
done
