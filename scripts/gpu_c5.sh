# C5 at its BASELINE parameters (flat facets, eps_ACA 1e-5, 64 RHS): parity test + timings
set -x
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k config5_flat > gpurun_out/pytest_c5.log 2>&1; echo c5test rc=$?
tail -5 gpurun_out/pytest_c5.log
timeout 900 python scripts/config_run.py 5 --rows 300 > gpurun_out/c5_flat.json 2> gpurun_out/c5_flat.err; echo c5run rc=$?
cat gpurun_out/c5_flat.json; tail -5 gpurun_out/c5_flat.err
