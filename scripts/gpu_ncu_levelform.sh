# ncu evidence for the pure level-form solve (cut = depth, 39 passes) on C2: the per-pass trace, then one
# --set full capture of the flux program (after the command exits 0 without ncu)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
CUT=99 timeout 300 python scripts/trace_step.py > gpurun_out/trace_levelform_c2.txt 2>&1; echo trace rc=$?
timeout 300 python scripts/prof_step.py --steps 1 --cut 99 > /dev/null 2>&1 && echo prof-ok
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:engine_kernel -c 1 \
  -o gpurun_out/prof_levelform -f python scripts/prof_step.py --steps 1 --cut 99 > gpurun_out/ncu_lf.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/prof_levelform.ncu-rep --page details > gpurun_out/levelform_full.txt 2>&1
