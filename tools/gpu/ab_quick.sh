# usage (under gpurun): bash tools/gpu/ab_quick.sh [rounds] -> quick GPU parity of the in-tree lib + A/B of ab/*.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_small or async or ragged or update_variants" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
bash tools/gpu/ab.sh ${1:-3}
