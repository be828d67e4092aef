python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "multi_rhs or host_pointers" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_shard.py -x -q --tb=short -k "multi_rhs" 2>&1 | tail -2
timeout 300 python scripts/mrhs_bench.py 2>&1 | tail -3
timeout 300 python scripts/mrhs_bench.py 4 2>&1 | tail -3
