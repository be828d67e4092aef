# evidence after the stage-geometry change: build, smoke, full GPU suite, bench, reference arm, ncu launch
# list of the bench command, one --set full capture of the engine (C2 flux step)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-level-form --profile-iters 2 > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 300 python scripts/prof_step.py --steps 1 > /dev/null 2>&1 && echo prof-ok
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:engine_kernel -c 1 \
  -o gpurun_out/prof_engine -f python scripts/prof_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
ncu -i gpurun_out/prof_engine.ncu-rep --page details > gpurun_out/engine_full.txt 2>&1
ncu -i gpurun_out/prof_engine.ncu-rep --page raw --csv > gpurun_out/engine_raw.csv 2>&1
