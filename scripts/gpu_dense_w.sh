# level form: W blocks of small nodes stored dense (HM_DENSE_W_ROWS; 0 = the previous rule) -- level-form
# parity tests with the default, then the cut-level sweep on C2 for several thresholds
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x \
  -k "solve_and_flux or level_form or hierarchical_and_dense or multi_rhs_level or fibonacci" 2>&1 | tail -2
for r in 0 160 320 640 1280; do
  echo "=== HM_DENSE_W_ROWS=$r"
  HM_DENSE_W_ROWS=$r CUTS=3,9 timeout 600 python scripts/cut_sweep.py 2>&1 | grep "^cut"
done
