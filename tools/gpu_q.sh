mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pair" 2>&1 | tail -1
b() { timeout 300 python bench.py --config $1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $3 > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],3),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
for i in 1 2; do b c4 base ""; LSP_APPLY_PAIR=1 b c4 pair ""; done
b c4-bf16 base ""; LSP_APPLY_PAIR=1 b c4-bf16 pair ""
for st in 3; do LSP_APPLY_STAGES=$st b c4 st$st ""; done
