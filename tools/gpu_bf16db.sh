# bf16 gather compress double-buffered (raw 16-byte segments): parity + bench C4-bf16, C3, C2, C4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -x -k "compress or bf16 or full_size" 2>&1 | tail -3
for c in c4-bf16 c3 c4; do
timeout 600 python bench.py --config $c --fit-every 0 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
python -c "
import json;d=json.load(open('gpurun_out/b_$c.json'));print('$c', round(d['ms_per_step'],3), d['breakdown']['compress_ms_per_step'], d['config']['step_hbm_frac_of_measured'])" || tail -3 gpurun_out/b_$c.err
done
