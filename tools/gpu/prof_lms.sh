# usage (under gpurun): bash tools/gpu/prof_lms.sh -> gpurun_out/prof_lms.ncu-rep
mkdir -p gpurun_out
python tools/prof_run.py C5 4 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kk_lms -s 1 -c 1 -o gpurun_out/prof_lms -f \
    python tools/prof_run.py C5 4 > gpurun_out/ncu_lms.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_lms.log
