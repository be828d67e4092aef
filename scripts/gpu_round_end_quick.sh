# round-end evidence without the GPU suite (scripts/gpu_suite_durations.sh runs that): smoke, bench, reference arm, ncu
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
( time timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver_cmd.json 2> gpurun_out/bench_driver_cmd.err ) 2>&1 | grep real; echo bench20 rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err ) 2>&1 | grep real; echo ref rc=$?
head -12 scripts/gpu_ncu.sh | tail -9 > /tmp/ncu_part.sh; bash /tmp/ncu_part.sh > gpurun_out/ncu_all.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/prof_engine.ncu-rep --page details > gpurun_out/engine_full.txt 2>&1
ncu -i gpurun_out/prof_engine.ncu-rep --page raw --csv > gpurun_out/engine_raw.csv 2>&1
rm -f gpurun_out/*.ncu-rep
