# usage (under gpurun): bash tools/gpu/prof_bench.sh TAG -> gpurun_out/prof_bench_chain_TAG.ncu-rep
# ncu --set full of the timed combined chain launch of the bench command (launch index 5, see evidence.sh)
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cufft"
timeout 300 $CMD > gpurun_out/bench_short_$1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kk_chain -s 5 -c 1 -o gpurun_out/prof_bench_chain_$1 -f $CMD > gpurun_out/ncu_full_$1.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full_$1.log
