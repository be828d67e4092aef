# multi-RHS engine variants (rebuilt with HM_BUILD_DEFINES): C2 64-RHS flux / apply / solve
for d in "" "HM_MRHS_GATHER_LDG=0"; do
  HM_BUILD_DEFINES="$d" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null || exit 1
  echo "== defines: [$d]"
  timeout 600 python scripts/mrhs_bench.py 2>&1 | grep -v "^\[hm\]"
done
python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null
