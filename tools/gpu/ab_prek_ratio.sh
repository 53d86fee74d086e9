# usage (under gpurun): bash tools/gpu/ab_prek_ratio.sh -> pre-KK ratio (tools/next_rows_bench.py row 3) per ab/*.so
mkdir -p gpurun_out
: > gpurun_out/ab_prek.log
for lib in ab/*.so; do
  KKRX_LIB=$lib timeout 600 python tools/next_rows_bench.py 64 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin)['row3_pre_kk_equaliser']; print('$lib', round(d['value_without'],2), round(d['value_with_15_taps'],2), round(d['ratio'],4))" >> gpurun_out/ab_prek.log
done
