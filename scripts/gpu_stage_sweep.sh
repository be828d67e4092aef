# engine stage-geometry experiment (C2): per variant, forced rebuild with HM_BUILD_DEFINES, a C2 parity
# subset, and the flux step time (bench without extras)
for v in "" "HM_PSTAGES=4 HM_STAGE_DOUBLES=5120" "HM_STAGE_DOUBLES=4320" "HM_GSLOTS=8 HM_RSLOTS=4" "HM_STAGE_DOUBLES=4608 HM_GSLOTS=8 HM_RSLOTS=4"; do
  echo "== variant [$v]"
  HM_BUILD_DEFINES="$v" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" || continue
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "config2_full_size or (solve_and_flux and C1)" 2>&1 | tail -1
  for r in 1 2; do
    timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --no-level-form 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('flux us', round(d['ms_per_step']*1e3,1), 'engine us', round(d['config']['engine_ms']['flux']*1e3,1), 'apply us', round(d['config']['engine_ms']['apply_F']*1e3,1), 'units', d['config']['engine']['units'], 'frac', round(d['roofline']['frac'],4))"
  done
done
python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)"
