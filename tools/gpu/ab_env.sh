# A/B of one library under two environments: bash tools/gpu/ab_env.sh LIB "ENV_A" "ENV_B" [rounds]
mkdir -p gpurun_out
R=${4:-3}
: > gpurun_out/ab.log
for r in $(seq 1 $R); do
  for e in "$2" "$3"; do
    env $e KKRX_LIB=$1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-cufft 2>>gpurun_out/ab.err | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({'env': '$e', 'value': round(d['value'],2), 'k': {k: round(v,4) for k,v in d['kernel_ms_per_step'].items()}}))" >> gpurun_out/ab.log
  done
done
