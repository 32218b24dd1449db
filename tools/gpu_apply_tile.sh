# Apply ring-tile experiment: C4 / C4-bf16 / C3 bench splits (+ stage count override).
mkdir -p gpurun_out
for c in c4 c4-bf16 c3; do
for stg in "" 8 6; do
LSP_APPLY_STAGES=${stg:-16} timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/at.json 2> gpurun_out/at.err
python -c "
import json;d=json.load(open('gpurun_out/at.json'));b=d['breakdown'];print('$c stages=${stg:-max}', round(d['ms_per_step'],3), 'apply', round(b['apply_ms_per_step'],3), 'build', round(b['build_y_ms_per_step'],3))" || tail -3 gpurun_out/at.err
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer.py tests/test_gpu_schedule.py -m gpu -x -q 2>&1 | tail -2
