# usage (under gpurun): bash tools/gpu/phase_timing.sh  (ab/t_timing.so built with -DKK_PHASE_TIMING=1)
mkdir -p gpurun_out
KKRX_PHASE_TIMING=1 KKRX_LIB=ab/t_timing.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cufft > gpurun_out/phase_timing.log 2>&1
KKRX_PHASE_TIMING=1 KKRX_LIB=ab/t_timing.so timeout 300 python tools/prof_run.py C5 4 >> gpurun_out/phase_timing.log 2>&1
