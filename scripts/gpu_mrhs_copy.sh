# multi-RHS engine copy paths (C2, 64 RHS): X-tile gather by 16-byte cp.async vs per-row TMA, and the
# payload of conflict-free chunks as one bulk copy vs per-column copies; per variant: multi-RHS parity
# tests, then flux / apply / solve timings
for d in "" "HM_MRHS_WHOLE_CHUNK=2"; do
  echo "=== variant: [$d]"
  HM_BUILD_DEFINES="$d" python -c "import __graft_entry__ as g; g.build()" > /dev/null || { echo build-failed; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "multi_rhs" 2>&1 | tail -1
  timeout 300 python scripts/mrhs_bench.py 2>&1 | tail -3
done
