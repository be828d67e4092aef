# multi-RHS engine stage-geometry sweep (C2, 64 RHS): X-tile columns / payload doubles / stages set at build
# time (HM_BUILD_DEFINES); per variant: the multi-RHS parity tests, then flux / apply / solve timings
for d in "" "HM_MRHS_MAXCOLS=64 HM_MRHS_PAYLOAD=2432 HM_MRHS_STAGES=4" "HM_MRHS_MAXCOLS=48 HM_MRHS_PAYLOAD=3072 HM_MRHS_STAGES=4" \
         "HM_MRHS_MAXCOLS=64 HM_MRHS_PAYLOAD=4608 HM_MRHS_STAGES=3"; do
  echo "=== variant: [$d]"
  HM_BUILD_DEFINES="$d" python -c "import __graft_entry__ as g; g.build()" > /dev/null || { echo build-failed; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "multi_rhs_dmma" 2>&1 | tail -1
  timeout 300 python scripts/mrhs_bench.py 2>&1 | tail -3
done
