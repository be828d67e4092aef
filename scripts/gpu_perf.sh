# perf iteration: build, parity, engine stats, cut sweep
python -c "import __graft_entry__ as g; g.build()"
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --tb=short 2>&1 | tail -15
HM_ENGINE_STATS=1 timeout 300 python scripts/engine_stats.py 2>&1 | grep -A1 "^---" | grep engine | awk 'NR%3==0' 
CUTS=0,9 timeout 300 python scripts/cut_sweep.py 2>&1 | tee gpurun_out/cut_pf.log
CUT=0 timeout 200 python scripts/trace_step.py 2>&1 | tail -12
