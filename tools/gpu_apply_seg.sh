# Apply unit length (row blocks per unit, LSP_APPLY_SEG): drift between adjacent-band CTAs vs Y reloads.
mkdir -p gpurun_out
for seg in 0 8 16 32; do
if [ $seg = 0 ]; then unset LSP_APPLY_SEG; else export LSP_APPLY_SEG=$seg; fi
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/sg.json 2> gpurun_out/sg.err
python -c "
import json;d=json.load(open('gpurun_out/sg.json'));b=d['breakdown'];print('seg=$seg', round(d['ms_per_step'],3), 'apply', round(b['apply_ms_per_step'],3), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sg.err
done
