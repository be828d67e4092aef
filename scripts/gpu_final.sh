# end-of-round evidence: build, smoke, full GPU suite, bench (+ reference arm), ncu launch list and full
# captures (engine + multi-RHS engine), full-size configs C3-C5
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
cat gpurun_out/bench_ref.json
bash scripts/gpu_ncu.sh
timeout 300 python scripts/mrhs_bench.py 2>&1 | tail -3
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:engine_mrhs -c 1 -o gpurun_out/prof_mrhs_final -f python scripts/prof_mrhs.py > gpurun_out/ncu_m_final.log 2>&1; echo ncu4 rc=$?
bash scripts/gpu_configs.sh
