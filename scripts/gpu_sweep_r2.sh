# stage geometry and piece sizing re-swept with the stage-B operators (C2 flux; two runs each)
run() { for r in 1 2; do timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --no-level-form 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('  flux us', round(d['ms_per_step']*1e3,1), 'engine us', round(d['config']['engine_ms']['flux']*1e3,1), 'units', d['config']['engine']['units'], 'frac', round(d['roofline']['frac'],4))"; done; }
for vv in _default HM_PSTAGES=4_HM_STAGE_DOUBLES=5424 HM_PSTAGES=2_HM_STAGE_DOUBLES=10860; do
  v="${vv//_HM/ HM}"; v="${v#_default}"
  echo "== stages [$v]"
  HM_BUILD_DEFINES="$v" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null || continue
  run
done
python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null
for cfg in "1 4" "4 4" "2 2" "2 8"; do
  set -- $cfg
  echo "== HM_PIECE_DIV=$1 HM_PIECE_MIN=$2"
  HM_PIECE_DIV=$1 HM_PIECE_MIN=$2 run
done
