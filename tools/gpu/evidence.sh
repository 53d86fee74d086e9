# Full evidence run (under gpurun): bench (with e2e + cpu_baseline), reference arm,
# ncu launch list of the bench command, ncu --set full of the timed combined chain launch.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cufft"
timeout 300 $CMD > gpurun_out/bench_short.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launches.log
# chain-kernel launches of $CMD: warm-up [tails(0)] [apply(0)+tails(1)] [apply(1)+tails(2)] [apply(2)],
# timed [tails(3)] [apply(3)+tails(4)] [apply(4)] -> index 5 is the timed combined launch
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kk_chain -s 5 -c 1 -o gpurun_out/prof_bench_chain -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kk_lms -s 1 -c 1 -o gpurun_out/prof_bench_lms -f $CMD > gpurun_out/ncu_full_lms.log 2>&1
echo "full lms rc=$?" >> gpurun_out/ncu_full_lms.log
