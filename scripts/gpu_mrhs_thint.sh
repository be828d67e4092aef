# multi-RHS engine: L2 policy of the phase-1 -> phase-2 scratch t (HM_MRHS_T_HINT), C2 64-RHS flux
for d in "" "HM_MRHS_T_HINT=1" "HM_MRHS_T_HINT=2" ""; do
  HM_BUILD_DEFINES="$d" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null || exit 1
  echo "== defines: [$d]"
  timeout 600 python scripts/mrhs_bench.py 2 64 20 2>&1 | grep -v "^\[hm\]"
done
