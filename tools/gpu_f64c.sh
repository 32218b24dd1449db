# fp64 Y path (apply_f64.cu): parity, every GPU test touching fp64 / decompress, C4-f64 and C4 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fit.py tests/test_gpu_layer.py tests/test_gpu_conformance.py -q -x 2>&1 | tail -4
timeout 1200 python bench.py --config c4-f64 --no-cpu-baseline > gpurun_out/bench_c4-f64.json 2> gpurun_out/bench_c4-f64.err
python -c "
import json;d=json.load(open('gpurun_out/bench_c4-f64.json'));print('c4-f64', round(d['ms_per_step'],3), round(d['value'],1), d['config']['step_hbm_frac_of_measured'], d['roofline']['frac'], d['breakdown'], d['e2e']['value'])" || tail -20 gpurun_out/bench_c4-f64.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c4.json 2>gpurun_out/c4.err; python -c "
import json;d=json.load(open('gpurun_out/c4.json'));print('c4', round(d['ms_per_step'],3), d['breakdown']['apply_ms_per_step'])"
