# multi-RHS engine variants (run-based X gather on/off): parity + timing + per-pass trace
for d in "" "HM_MRHS_X_RUNS=0"; do
  echo "=== variant: [$d]"
  HM_BUILD_DEFINES="$d" python -c "import __graft_entry__ as g; g.build()" > /dev/null || { echo build-failed; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "multi_rhs" 2>&1 | tail -1
  timeout 300 python scripts/mrhs_bench.py 2>&1 | tail -3
  HM_TRACE_MRHS=1 timeout 300 python scripts/mrhs_stats.py 2>&1 | grep "trace" | tail -8
done
