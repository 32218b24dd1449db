# Sweep the gather-compress L2 prefetch distance (LSP_SPMM_PF column tiles; 0 = off).
mkdir -p gpurun_out
for pf in ${1:-0 8 12 16 24 32}; do
  LSP_SPMM_PF=$pf timeout 300 python bench.py --config ${2:-c4} --no-e2e --no-cpu-baseline > gpurun_out/pf.json 2> gpurun_out/pf.err
  python -c "
import json;d=json.load(open('gpurun_out/pf.json'));b=d['breakdown'];print('pf=$pf', 'ms/step',round(d['ms_per_step'],2),'compress',round(b['compress_ms_per_step'],2))" || tail -2 gpurun_out/pf.err
done
