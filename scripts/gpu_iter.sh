# build, parity suite (incl. C2 full size), bench; used for each optimisation iteration
timeout 150 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
HM_DEBUG=1 timeout 420 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
timeout 240 python bench.py --steps 100 --warmup 10 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python - <<'P'
import json
d = json.load(open("gpurun_out/bench.json"))
c = d["config"]
print("applies/s %.1f  ms/step %.4f  step GB/s %.0f (%.1f%%)  e2e %.1f" % (d["value"], d["ms_per_step"], c["step_hbm_gbs"], 100*c["step_frac_of_peak"], d["e2e"]["value"]))
print("engine_ms", c["engine_ms"], c["engine"], "F GB/s %.0f  C GB/s %.0f" % (c["apply_F_hbm_gbs"], c["solve_C_hbm_gbs"]))
print("roofline", d["roofline"])
print("bytes F %.1f MB C %.1f MB ranksC %s clocks %s" % (c["bytes_F"]/1e6, c["bytes_C"]/1e6, c["ranks_C"], d["clocks"]))
P
tail -3 gpurun_out/bench.err
timeout 120 python scripts/trace_step.py 2>&1 | tail -60
timeout 300 python scripts/cut_sweep.py 2>&1 | tail -12
