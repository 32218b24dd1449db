mkdir -p gpurun_out/part
run() {  # tag, args...
  tag=$1; shift
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
    > gpurun_out/part/$tag.json 2> gpurun_out/part/$tag.err
  python -c "
import json
d=json.load(open('gpurun_out/part/$tag.json'))
print('%-12s step %.2f  part %s' % ('$tag', d['ms_per_step'], d['config'].get('partition_sms')))" || tail -4 gpurun_out/part/$tag.err
}
run base
for k in 56 64 72 80; do LSP_PART_STAGE2=1 run s2c_p$k --partition $k; done
run bf16_base --config c4-bf16
for k in 56 64 72; do run bf16_p$k --config c4-bf16 --partition $k; done
for k in 64 72; do LSP_PART_STAGE2=1 run bf16_s2c_p$k --config c4-bf16 --partition $k; done
run c3_base --config c3 --fit-every 0
for k in 48 56 64; do run c3_p$k --config c3 --fit-every 0 --partition $k; done
