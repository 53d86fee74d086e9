mkdir -p gpurun_out
python tools/prof_run.py C5 4 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kk_x2 -s 1 -c 1 -o gpurun_out/prof_x2 python tools/prof_run.py C5 4 > gpurun_out/ncu_x2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_x2.log
