for t in 16 8 4; do
  sed -i "s/    if (TM > [0-9]* \&\& 8 % N8 == 0) {/    if (TM > $t \&\& 8 % N8 == 0) {/" paper_2305_06891_b200/csrc/kernels_mrhs.cu
  python -c "import paper_2305_06891_b200.build as b; b.build(force=True)" > /dev/null 2>&1 || { echo build fail; continue; }
  echo "== prefetch for TM <= $t"; timeout 300 python scripts/mrhs_bench.py 2>&1 | tail -3
done
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "multi_rhs" 2>&1 | tail -2
