# stage-geometry candidates on the large configs: C4 F apply (1 vector) and C3 flux
for vv in _default HM_PSTAGES=4_HM_STAGE_DOUBLES=5432 HM_PSTAGES=3_HM_STAGE_DOUBLES=7240; do
  v="${vv//_HM/ HM}"; v="${v#_default}"
  echo "== variant [$v]"
  HM_BUILD_DEFINES="$v" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" || continue
  timeout 600 python scripts/config_run.py 4 --rows 50 --nrhs 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('C4 apply ms', round(d['apply_ms'],3), 'GB/s', round(d['apply_GBs']), 'rel', d['apply_sampled_rel'])"
  timeout 900 python scripts/config_run.py 3 --rows 50 --nrhs 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('C3 apply ms', round(d['apply_ms'],3), 'flux ms', round(d['flux_ms'],3), 'flux GB/s', round(d['flux_GBs']), 'resid', d['solve_sampled_resid_rel'])"
done
