# perf iteration: build, quick parity, per-pass trace and cut sweep (with / without the L2 prefetch warp)
python -c "import __graft_entry__ as g; g.build()"
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
CUT=0 timeout 200 python scripts/trace_step.py > gpurun_out/trace0.log 2>&1
CUTS=0,2,9 timeout 300 python scripts/cut_sweep.py 2>&1 | tee gpurun_out/cut_pf.log
HM_PREFETCH=0 CUTS=0,9 timeout 300 python scripts/cut_sweep.py 2>&1 | tee gpurun_out/cut_nopf.log
