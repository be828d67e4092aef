set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k config2 2>&1 | tail -5
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$?
cat gpurun_out/bench1.json
tail -5 gpurun_out/bench1.err
