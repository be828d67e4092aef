# multi-RHS programs: element-wise epilogue pass (default) vs emit from the last stream pass (HM_MRHS_FUSED_EPI=1)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for v in 0 1 0 1; do
  echo "== HM_MRHS_FUSED_EPI=$v"
  HM_MRHS_FUSED_EPI=$v timeout 600 python scripts/mrhs_bench.py 2 64 20 2>&1 | grep -v "^\[hm\]"
done
HM_MRHS_FUSED_EPI=1 timeout 600 python scripts/mrhs_bench.py 3 64 10 2>&1 | grep -v "^\[hm\]"
HM_MRHS_FUSED_EPI=0 timeout 600 python scripts/mrhs_bench.py 3 64 10 2>&1 | grep -v "^\[hm\]"
HM_MRHS_FUSED_EPI=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "multi_rhs or exported or config2" 2>&1 | tail -3
