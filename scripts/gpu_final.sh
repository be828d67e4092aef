# end-of-round evidence: smoke, full GPU suite (with a host-memory trace), bench (+ reference arm), ncu
# launch list and one --set full capture of the engine (each ncu run after its command exits 0 without ncu)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke.log
( while true; do echo "$(date +%s) $(free -g | head -2 | tail -1)" >> gpurun_out/mem_final.log; sleep 15; done ) & MP=$!
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
kill $MP
tail -32 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
cat gpurun_out/bench_ref.json
bash scripts/gpu_ncu.sh > gpurun_out/ncu_all.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/prof_engine.ncu-rep --page details > gpurun_out/engine_full.txt 2>&1
ncu -i gpurun_out/prof_engine.ncu-rep --page raw --csv > gpurun_out/engine_raw.csv 2>&1
