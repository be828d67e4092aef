python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python scripts/config_run.py 3 --nrhs 64 > gpurun_out/c3.json 2> gpurun_out/c3.err; echo c3 rc=$?; tail -c 1500 gpurun_out/c3.json
timeout 900 python scripts/config_run.py 4 --nrhs 64 --rows 300 > gpurun_out/c4.json 2> gpurun_out/c4.err; echo c4 rc=$?; tail -c 1500 gpurun_out/c4.json
timeout 900 python scripts/config_run.py 5 --exact --nrhs 64 --rows 300 > gpurun_out/c5x.json 2> gpurun_out/c5x.err; echo c5 rc=$?; tail -c 1500 gpurun_out/c5x.json
