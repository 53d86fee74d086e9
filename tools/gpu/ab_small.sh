mkdir -p gpurun_out; : > gpurun_out/ab_small.log
for lib in ab/a_head.so ab/b_lms2.so ab/a_head.so ab/b_lms2.so; do
  for b in 4 16 128; do
    KKRX_LIB=$lib timeout 300 python bench.py --batch $b --steps 20 --no-cpu-baseline --no-cufft --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$lib', $b, round(d['value'],2), round(d['sync_value'],2), round(d['kernel_ms_per_step']['lms_overlapped'],4))" >> gpurun_out/ab_small.log
  done
done
