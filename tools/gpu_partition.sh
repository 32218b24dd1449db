# Partitioned step (lsp_schedule_set_partition): green-context SM split between
# the stage-1 chain and the update chain, C4 fp32 (and bf16 / C3), vs serial.
mkdir -p gpurun_out/part
run() {  # tag, args...
  tag=$1; shift
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
    > gpurun_out/part/$tag.json 2> gpurun_out/part/$tag.err
  python -c "
import json
d=json.load(open('gpurun_out/part/$tag.json'))
print('%-12s step %.2f  part %s graph %s' % ('$tag', d['ms_per_step'], d['config'].get('partition_sms'), bool(d['config']['cuda_graph'])))" || tail -4 gpurun_out/part/$tag.err
}
run base
for k in 48 56 64 72 80; do run p$k --partition $k; done
run p64_g0 --partition 64 --graph 0
