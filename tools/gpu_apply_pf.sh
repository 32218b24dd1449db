# Apply L2 prefetch distance (LSP_APPLY_PF tiles ahead of the 10-stage ring), C4 and C4-bf16.
mkdir -p gpurun_out
for c in c4 c4-bf16; do for pf in 0 14 20 32; do
LSP_APPLY_PF=$pf timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/pf.json 2> gpurun_out/pf.err
python -c "
import json;d=json.load(open('gpurun_out/pf.json'));b=d['breakdown'];print('$c pf=$pf', round(d['ms_per_step'],3), 'apply', round(b['apply_ms_per_step'],3))" || tail -3 gpurun_out/pf.err
done; done
