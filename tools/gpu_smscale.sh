# Phase times vs SM budget (lsp_set_sm_budget), C4 fp32: does the apply keep its
# HBM rate on fewer SMs, and how does compress scale?  Then the two-stream
# (compress chain / update chain) schedule under complementary budgets.
mkdir -p gpurun_out/smscale
run() {  # tag, args...
  tag=$1; shift
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
    > gpurun_out/smscale/$tag.json 2> gpurun_out/smscale/$tag.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/smscale/$tag.json')); b=d['breakdown']
print('%-14s step %.2f  compress %.2f adam %.2f build %.2f apply %.2f' % ('$tag', d['ms_per_step'], b['compress_ms_per_step'], b['adam_ms_per_step'], b['build_y_ms_per_step'], b['apply_ms_per_step']))" || tail -2 gpurun_out/smscale/$tag.err
}
run base
for k in 128 112 96 80 64; do run u$k --sms-update $k; done
for k in 112 96 74; do run c$k --sms-compress $k; done
run conc --concurrent 1 --schedule python
for kc in 48 64 74; do run conc_c${kc} --concurrent 1 --schedule python --sms-compress $kc --sms-update $((148 - kc)); done
