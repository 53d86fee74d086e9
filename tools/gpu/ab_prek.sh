# usage (under gpurun): bash tools/gpu/ab_prek.sh -> pre-KK parity + NEXT-rows bench + A/B of ab/*.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pre_kk or parity_small or async" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python tools/next_rows_bench.py 64 > gpurun_out/next_rows.json 2> gpurun_out/next_rows.err; echo "next rc=$?" >> gpurun_out/next_rows.err
bash tools/gpu/ab.sh 3
