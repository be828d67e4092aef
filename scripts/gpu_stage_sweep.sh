# two payload stages of 85 KB vs the adopted three of 56.6 KB (C2 flux)
for vv in _default HM_PSTAGES=2_HM_STAGE_DOUBLES=10860; do
  v="${vv//_HM/ HM}"; v="${v#_default}"
  echo "== variant [$v]"
  HM_BUILD_DEFINES="$v" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null || continue
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "config2_full_size or (solve_and_flux and C1)" 2>&1 | tail -1
  for r in 1 2; do
    timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --no-level-form 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('flux us', round(d['ms_per_step']*1e3,1), 'engine us', round(d['config']['engine_ms']['flux']*1e3,1), 'units', d['config']['engine']['units'], 'frac', round(d['roofline']['frac'],4))"
  done
done
