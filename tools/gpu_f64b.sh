# fp64 gather-form stage 1: parity (bitwise vs the CSC-walk kernel, 1e-12 vs the oracle), fp32 paths unchanged, C4-f64 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "compress_paths or slots_value or full_size or determinism" 2>&1 | tail -3
timeout 1200 python bench.py --config c4-f64 --no-cpu-baseline > gpurun_out/bench_c4-f64.json 2> gpurun_out/bench_c4-f64.err
python -c "
import json;d=json.load(open('gpurun_out/bench_c4-f64.json'));print('c4-f64', round(d['ms_per_step'],3), round(d['value'],1), d['config']['step_hbm_frac_of_measured'], d['breakdown'], d['e2e']['value'])" || tail -20 gpurun_out/bench_c4-f64.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c4.json 2>gpurun_out/c4.err; python -c "
import json;d=json.load(open('gpurun_out/c4.json'));print('c4', round(d['ms_per_step'],3), d['breakdown']['compress_ms_per_step'])"
