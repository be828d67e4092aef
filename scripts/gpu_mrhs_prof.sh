# multi-RHS engine evidence (C2, 64 RHS flux): per-role cycle counters, per-pass trace, one ncu --set full
# capture with source correlation (each after its own command exits 0 without ncu)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
HM_ENGINE_STATS=1 HM_TRACE_MRHS=1 timeout 600 python scripts/mrhs_stats.py > gpurun_out/mrhs_stats.log 2>&1; echo stats rc=$?
timeout 600 python scripts/mrhs_bench.py > gpurun_out/mrhs_bench.log 2>&1; echo mbench rc=$?
timeout 300 python scripts/prof_mrhs.py > /dev/null 2>&1 && echo prof-ok
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:engine_mrhs_kernel -c 1 \
  -o gpurun_out/prof_mrhs -f python scripts/prof_mrhs.py > gpurun_out/ncu_mrhs.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/prof_mrhs.ncu-rep --page details > gpurun_out/mrhs_full.txt 2>&1
ncu -i gpurun_out/prof_mrhs.ncu-rep --page source --csv > gpurun_out/mrhs_source.csv 2>&1
ncu -i gpurun_out/prof_mrhs.ncu-rep --page raw --csv > gpurun_out/mrhs_raw.csv 2>&1
