# the whole GPU suite under the default session time budget (tests/conftest.py), with per-test durations
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=45 -rs > gpurun_out/pytest_budget.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_budget.log
( time timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err ) 2> gpurun_out/bench_time.txt; echo bench rc=$?
cat gpurun_out/bench_time.txt
