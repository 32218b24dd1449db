# Native pipelined schedule: tests + bench per config (auto pipeline per W dtype).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_comm_overlap.py tests/test_gpu_schedule.py -m gpu -q -x 2>&1 | tail -1
for c in c4 c4-bf16 c3 c2; do
timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/pp.json 2> gpurun_out/pp.err
python -c "
import json;d=json.load(open('gpurun_out/pp.json'));print('$c', round(d['ms_per_step'],3), d['config']['schedule'][:6], d['config']['pipeline'])" || tail -3 gpurun_out/pp.err
done
for c in c4-bf16 c3 c2; do
timeout 600 python bench.py --config $c --pipeline 0 --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/pp.json 2> gpurun_out/pp.err
python -c "
import json;d=json.load(open('gpurun_out/pp.json'));print('$c pipeline=0', round(d['ms_per_step'],3))" || tail -3 gpurun_out/pp.err
done
