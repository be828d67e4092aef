# multi-RHS engine payload copy route (C2, 64 RHS): one bulk copy per chunk (HM_MRHS_WHOLE_CHUNK=2, default),
# only the conflict-free chunks whole (=1), every chunk column by column at a padded stride (=0); per
# variant: multi-RHS parity tests, then flux / apply / solve timings.  (This session's sweeps also measured
# cp.async gathers / payloads and an unpadded run-copied X tile; those code paths were removed.)
for d in "" "HM_MRHS_WHOLE_CHUNK=1" "HM_MRHS_WHOLE_CHUNK=0"; do
  echo "=== variant: [$d]"
  HM_BUILD_DEFINES="$d" python -c "import __graft_entry__ as g; g.build()" > /dev/null || { echo build-failed; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "multi_rhs" 2>&1 | tail -1
  timeout 300 python scripts/mrhs_bench.py 2>&1 | tail -3
done
