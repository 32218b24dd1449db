# Stage-2 matrix order: reverse (default) vs forward.
mkdir -p gpurun_out
for c in c4 c4-bf16; do for v in 1 0; do
LSP_STAGE2_REVERSE=$v timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/s2.json 2> gpurun_out/s2.err
python -c "
import json;d=json.load(open('gpurun_out/s2.json'));b=d['breakdown'];print('$c rev=$v', round(d['ms_per_step'],3), 'compress', round(b['compress_ms_per_step'],3))" || tail -3 gpurun_out/s2.err
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer.py -m gpu -x -q 2>&1 | tail -1
