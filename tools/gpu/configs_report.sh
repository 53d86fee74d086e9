# usage (under gpurun): bash tools/gpu/configs_report.sh -> full-size config tests + C1-C5 report at the stated sizes
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -s -k "full_size or c4_hdfec" > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
timeout 2400 python tests/reports/run_configs.py --out gpurun_out/configs_report.json > gpurun_out/configs_report.log 2>&1; echo "report rc=$?" >> gpurun_out/configs_report.log
