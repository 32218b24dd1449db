# FFMA2/FMUL2 in the gather compress and the apply consumers: bitwise tests + bench splits.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer.py tests/test_gpu_schedule.py tests/test_gpu_baseline_configs.py -m gpu -x -q 2>&1 | tail -2
for c in c4 c4-bf16 c3 c2; do
timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/f2.json 2> gpurun_out/f2.err
python -c "
import json;d=json.load(open('gpurun_out/f2.json'));b=d['breakdown'];print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in b.items() if k.endswith('per_step')})" || tail -3 gpurun_out/f2.err
done
