# A/B timing of library variants (under gpurun): bash tools/gpu/ab.sh [rounds]
# runs bench.py with each ab/*.so (KKRX_LIB) alternately; one JSON summary line per run in gpurun_out/ab.log
mkdir -p gpurun_out
R=${1:-3}
: > gpurun_out/ab.log
for r in $(seq 1 $R); do
  for lib in ab/*.so; do
    KKRX_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cufft 2>>gpurun_out/ab.err | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({'lib': '$lib', 'value': round(d['value'],2), 'k': {k: round(v,4) for k,v in d['kernel_ms_per_step'].items()}}))" >> gpurun_out/ab.log
  done
done
