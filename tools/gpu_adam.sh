# Adam with two vectors in flight per thread: parity tests + C4 / C4-bf16 / C3 Adam phase.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer.py -m gpu -q -x 2>&1 | tail -1
for c in c4 c4-bf16 c3; do
timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/ad.json 2> gpurun_out/ad.err
python -c "
import json;d=json.load(open('gpurun_out/ad.json'));b=d['breakdown'];print('$c', round(d['ms_per_step'],3), 'adam', round(b['adam_ms_per_step'],3))" || tail -3 gpurun_out/ad.err
done
