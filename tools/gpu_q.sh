mkdir -p gpurun_out
b() { timeout 300 python bench.py --config $1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $3 > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],3), 'compress', round(b['compress_ms_per_step'],3))" || tail -3 gpurun_out/b.err; }
b c4 base ""
for pf in 0 1 2 4 8; do LSP_SPMM_PF=$pf b c4 pf$pf ""; done
