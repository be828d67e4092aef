# C5-size parity tests with a host-memory trace (the H-LU's host peak), then the multi-RHS tiling variants
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
( while true; do echo "$(date +%s) $(free -g | head -2 | tail -1)" >> gpurun_out/mem.log; sleep 10; done ) & MP=$!
HM_HLU_VERBOSE=1 timeout 2400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --durations=10 \
  -k "sphere_exact_solve or config5_flat or config4_apply" > gpurun_out/pytest_c5.log 2>&1; echo pytest rc=$?
kill $MP
grep -v "^\[hm\]\|^  " gpurun_out/pytest_c5.log | tail -25
grep "^\[hm\]" gpurun_out/pytest_c5.log
timeout 600 python scripts/mrhs_bench.py > gpurun_out/mrhs_bench_1d.log 2>&1; echo mb1 rc=$?; cat gpurun_out/mrhs_bench_1d.log
HM_BUILD_DEFINES="HM_MRHS_TILE1D=0" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null
timeout 600 python scripts/mrhs_bench.py > gpurun_out/mrhs_bench_2d.log 2>&1; echo mb2 rc=$?; cat gpurun_out/mrhs_bench_2d.log
python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null
