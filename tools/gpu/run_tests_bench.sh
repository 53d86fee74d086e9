# usage (under gpurun): bash tools/gpu/run_tests_bench.sh [ncu]
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ "$1" = "ncu" ]; then
  python tools/prof_run.py C5 4 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:kk_chain -s 3 -c 1 -o gpurun_out/prof_chain \
      python tools/prof_run.py C5 4 > gpurun_out/ncu_chain.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_chain.log
fi
