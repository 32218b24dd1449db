mkdir -p gpurun_out
b() { timeout 300 python bench.py --config $1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $3 > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],3), 'apply', round(b['apply_ms_per_step'],3))" || tail -3 gpurun_out/b.err; }
for seg in 48 64 128; do LSP_APPLY_SEG=$seg b c4 seg$seg ""; done
b c4 base ""
for seg in 64; do LSP_APPLY_SEG=$seg b c4-bf16 seg$seg ""; done
b c4-bf16 base ""
