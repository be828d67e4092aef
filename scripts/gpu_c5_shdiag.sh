# C5 flat with the 3-stage engine; then which sharded segment faults with stage-sized chunks (HM_DEBUG
# syncs after every launch and names it)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python scripts/config_run.py 5 --rows 100 > gpurun_out/c5_flat3.json 2> gpurun_out/c5_flat3.err; echo c5 rc=$?
cat gpurun_out/c5_flat3.json
HM_BUILD_DEFINES="HM_SHARD_CHUNK_UNCAPPED=1" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null
HM_DEBUG=1 timeout 300 python -m pytest tests/test_gpu_shard.py -x -q -k "match_single_rank_and_oracle and 2" > gpurun_out/shdiag.log 2>&1; echo shdiag rc=$?
grep -m 6 -E "HM_ERR|illegal|error|rank" gpurun_out/shdiag.log | cut -c1-400
python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null
