# GPU check of the oracle-H-LU parity test (all five parity cases) + smoke
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "hlu_factors_match_oracle or apply_equals_oracle" > gpurun_out/pytest_hlu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_hlu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
