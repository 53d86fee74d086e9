KKRX_EVENT_TRACE=1 timeout 300 python bench.py --batch 256 --steps 6 --no-cpu-baseline --no-cufft --no-e2e > gpurun_out/trace.log 2>&1
