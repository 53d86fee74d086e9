# usage (under gpurun): bash tools/gpu/race_jitter.sh [rounds]
# Race hunting without compute-sanitizer (closed on this pool): ab/jitter.so is the library
# built with -DKK_JITTER=1 (every warp sleeps a pseudo-random 0..4 us before each group barrier,
# tools/ab_build.py); its outputs must be bit-identical to the plain build's under many
# scrambled schedules, and it must still pass the oracle parity tests.
mkdir -p gpurun_out
R=${1:-5}
: > gpurun_out/race_jitter.log
timeout 300 python tools/sanitize_run.py 64 gpurun_out/labels_plain.npy >> gpurun_out/race_jitter.log 2>&1
for r in $(seq 1 $R); do
  KKRX_LIB=ab/jitter.so timeout 300 python tools/sanitize_run.py 64 gpurun_out/labels_jitter_$r.npy >> gpurun_out/race_jitter.log 2>&1
  python -c "import numpy as np,sys; a=np.load('gpurun_out/labels_plain.npy'); b=np.load('gpurun_out/labels_jitter_$r.npy'); print('round $r: jittered labels == plain build:', bool((a==b).all()), a.size)" >> gpurun_out/race_jitter.log 2>&1
done
KKRX_LIB=ab/jitter.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_small or async or ragged or update_variants or sharding or pre_kk" >> gpurun_out/race_jitter.log 2>&1
echo "jitter pytest rc=$?" >> gpurun_out/race_jitter.log
rm -f gpurun_out/labels_*.npy
