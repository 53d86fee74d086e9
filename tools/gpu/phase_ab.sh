# usage (under gpurun): bash tools/gpu/phase_ab.sh ab/t_X.so ...  (libraries built with -DKK_PHASE_TIMING=1)
mkdir -p gpurun_out
: > gpurun_out/phase_ab.log
for L in "$@"; do
  echo "== $L" >> gpurun_out/phase_ab.log
  KKRX_PHASE_TIMING=1 KKRX_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cufft 2>&1 | grep -E "PHASE|value" | cut -c1-220 >> gpurun_out/phase_ab.log
done
