mkdir -p gpurun_out
b() { timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],2),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
b c4 base
for mb in 40 64 96; do LSP_COMPRESS_ZT_MB=$mb b c4 zt$mb; done
LSP_COMPRESS_ZT_MB=64 b c4-bf16 zt64
b c4-bf16 base
