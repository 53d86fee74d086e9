# usage (under gpurun): bash tools/gpu/round_check.sh -> race-jitter check, smoke, pytest -m gpu, full evidence set
mkdir -p gpurun_out
bash tools/gpu/race_jitter.sh 5
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash tools/gpu/evidence.sh
