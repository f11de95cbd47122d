# Row-pass time of the SELL knob across kernel variants (tools/build_variants.sh) and CTAs per SM.
run() {  # label, env...
  local label=$1; shift
  env "$@" python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c1 --ttt-limit 2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$label', round(d['value'],1), {k:round(v['mean_us'],1) for k,v in d['roofline']['per_kernel'].items()}, d['clocks']['sm_mhz'])"
}
run base PDLP_X=0
run sell_default PDLP_ROW_SELL=1
run sell_ctas6 PDLP_ROW_SELL=1 PDLP_SELL_CTAS=6
run sell_ctas8 PDLP_ROW_SELL=1 PDLP_SELL_CTAS=8
run s3u8 PDLP_ROW_SELL=1 PDLP_SELL_CTAS=3 PDLP_LIB=$PWD/tools/variants/s3u8/libpdlp_b200.so
run s4u4 PDLP_ROW_SELL=1 PDLP_LIB=$PWD/tools/variants/s4u4/libpdlp_b200.so
run s6u4 PDLP_ROW_SELL=1 PDLP_SELL_CTAS=6 PDLP_LIB=$PWD/tools/variants/s6u4/libpdlp_b200.so
run s6u4_12 PDLP_ROW_SELL=1 PDLP_SELL_CTAS=12 PDLP_LIB=$PWD/tools/variants/s6u4/libpdlp_b200.so
