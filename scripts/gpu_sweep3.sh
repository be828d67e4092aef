python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for t in 4 16 64 100000; do
  echo "== mrhs piece min $t chunks"; HM_MRHS_PIECE_MIN=$t timeout 300 python scripts/mrhs_bench.py 2>&1 | tail -3
done
