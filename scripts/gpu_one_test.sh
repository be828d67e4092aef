# one GPU test with a host-memory trace: bash scripts/gpu_one_test.sh <pytest -k expression>
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
( while true; do echo "$(date +%s) $(free -g | head -2 | tail -1)" >> gpurun_out/mem_one.log; sleep 5; done ) & MP=$!
HM_HLU_VERBOSE=1 timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=5 -k "$1" > gpurun_out/pytest_one.log 2>&1; echo pytest rc=$?
kill $MP
grep -v "^  " gpurun_out/pytest_one.log | tail -30
awk '{print $4}' gpurun_out/mem_one.log | tr '\n' ' '
