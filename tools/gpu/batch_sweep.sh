# usage (under gpurun): bash tools/gpu/batch_sweep.sh -> gpurun_out/batch_sweep.jsonl
# streaming (and synchronous) GSa/s per batch size, device-resident, C5
mkdir -p gpurun_out
: > gpurun_out/batch_sweep.jsonl
for b in 4 8 16 32 48 64 96 128 256; do
  timeout 300 python bench.py --batch $b --steps 20 --no-cpu-baseline --no-cufft --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({'buffers_per_step': $b, 'value': round(d['value'],2), 'sync_value': round(d['sync_value'],2), 'chain_ms': round(d['kernel_ms_per_step']['chain'],4), 'ms_per_step': round(d['ms_per_step'],4), 'sm_mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/batch_sweep.jsonl
done
