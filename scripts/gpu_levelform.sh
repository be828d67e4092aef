# level-form solve: reader/writer tree dependencies (default) vs the conservative nearest-ancestor rule
# (HM_DEP_REFINED=0): level-form parity tests (single vector, 64 RHS, virtual shards, bitwise repeat),
# then the flux / solve time per cut level on C2 with both rules
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x \
  -k "solve_and_flux or level_form or hierarchical_and_dense or multi_rhs_level or fibonacci" 2>&1 | tail -3
for r in 1 0; do
  echo "=== HM_DEP_REFINED=$r"
  HM_DEP_REFINED=$r CUTS=0,1,2,3,9 timeout 600 python scripts/cut_sweep.py 2>&1 | grep "^cut"
done
