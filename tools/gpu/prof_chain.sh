# usage (under gpurun): bash tools/gpu/prof_chain.sh [tag] -> gpurun_out/prof_chain[_tag].ncu-rep
mkdir -p gpurun_out
T=${1:+_$1}
python tools/prof_run.py C5 4 > gpurun_out/prof_plain$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kk_chain -s 3 -c 1 -o gpurun_out/prof_chain$T -f \
    python tools/prof_run.py C5 4 > gpurun_out/ncu_chain$T.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_chain$T.log
