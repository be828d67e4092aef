# parity + bench + ncu launch list + one full ncu capture of the stream kernel
bash scripts/gpu_iter.sh
python scripts/prof_step.py --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python scripts/prof_step.py --steps 2 > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
python scripts/prof_step.py --steps 1 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:stream_kernel -c 4 \
    -o gpurun_out/prof_stream python scripts/prof_step.py --steps 1 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu2.log
