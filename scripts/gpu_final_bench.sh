# final-HEAD evidence without the full suite: the level-form / multi-RHS / flux parity subsets, bench (+ the
# reference arm), the ncu launch list of the bench command and one --set full capture of the engine
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -p no:cacheprovider \
  -k "solve_and_flux or level_form or multi_rhs or hierarchical_and_dense or exported_factors or config2" > gpurun_out/pytest_subset.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_subset.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
bash scripts/gpu_ncu.sh > gpurun_out/ncu_all.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/prof_engine.ncu-rep --page details > gpurun_out/engine_full.txt 2>&1
ncu -i gpurun_out/prof_engine.ncu-rep --page raw --csv > gpurun_out/engine_raw.csv 2>&1
