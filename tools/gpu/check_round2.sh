# usage (under gpurun): bash tools/gpu/check_round2.sh -> smoke, pytest -m gpu, bench (default + strong scaling)
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --scaling strong --steps 3 --no-e2e --no-cpu-baseline --no-cufft > gpurun_out/bench_strong.log 2>&1; echo "strong rc=$?" >> gpurun_out/bench_strong.log
