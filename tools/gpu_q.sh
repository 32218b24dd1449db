mkdir -p gpurun_out
timeout 700 python tools/dbg_pair.py 2>&1 | tail -12
b() { timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],2),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
b c4 base
LSP_APPLY_PAIR=1 b c4 pair
LSP_APPLY_PAIR=1 LSP_APPLY_STAGES=5 b c4 pairS5
LSP_APPLY_PAIR=1 b c4-bf16 pair
b c4-bf16 base
