# ncu evidence for profiles/: launch list of the bench command + one full capture of the engine and the
# multi-RHS engine (each after its own command exits 0 without ncu)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-level-form --profile-iters 2 > gpurun_out/b_plain.json 2>/dev/null && echo bench-ok
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-level-form --profile-iters 2 > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 300 python scripts/prof_step.py --steps 1 > /dev/null 2>&1 && echo prof-ok
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:engine_kernel -c 1 \
  -o gpurun_out/prof_engine -f python scripts/prof_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 300 python scripts/prof_mrhs.py > /dev/null 2>&1 && echo profm-ok
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none --csv \
  --log-file gpurun_out/mrhs_launch.csv python scripts/prof_mrhs.py > gpurun_out/ncu_m.log 2>&1; echo ncu3 rc=$?
