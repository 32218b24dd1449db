# Apply band width: BN = 32 (default) vs LSP_APPLY_BN=16 (64 KB Y block, deeper ring).
mkdir -p gpurun_out
for c in c4 c4-bf16 c3; do
for bn in 32 16; do
LSP_APPLY_BN=$bn timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/at.json 2> gpurun_out/at.err
python -c "
import json;d=json.load(open('gpurun_out/at.json'));b=d['breakdown'];print('$c bn=$bn', round(d['ms_per_step'],3), 'apply', round(b['apply_ms_per_step'],3), 'build', round(b['build_y_ms_per_step'],3))" || tail -3 gpurun_out/at.err
done; done
