mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer.py -q -x 2>&1 | tail -1
b() { timeout 300 python bench.py --config $1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $3 > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],3), 'build', round(b['build_y_ms_per_step'],3))" || tail -3 gpurun_out/b.err; }
b c4 sent ""; b c3 sent ""; b c4-bf16 sent ""
