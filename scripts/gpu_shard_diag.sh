# sharded path with the 3 x 56.6 KB stages: memcheck of one virtual-shard test, then the chunk cap variant
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 500 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_shard.py -x -q -k "match_single_rank_and_oracle and 2" > gpurun_out/memcheck_shard.log 2>&1; echo memcheck rc=$?
grep -m 12 -E "Invalid|at |by thread|Address|ERROR SUMMARY|passed|failed" gpurun_out/memcheck_shard.log
HM_BUILD_DEFINES="HM_SHARD_CHUNK_CAP=1" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null
timeout 600 python -m pytest tests/test_gpu_shard.py -q -x 2>&1 | tail -3
