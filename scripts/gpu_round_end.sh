# round-end evidence on one B200: full GPU suite, bench (+ reference arm), ncu launch list and full capture
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
bash scripts/gpu_ncu.sh > gpurun_out/ncu_all.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/prof_engine.ncu-rep --page details > gpurun_out/engine_full.txt 2>&1
ncu -i gpurun_out/prof_engine.ncu-rep --page raw --csv > gpurun_out/engine_raw.csv 2>&1
rm -f gpurun_out/*.ncu-rep
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_full.log
