mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "decompress or step or layer" 2>&1 | tail -2
b() { timeout 600 python bench.py --config $1 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],2),'frac',round(d['roofline']['frac'],3),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
b c4-bf16 x; b c3 x; b c4 x
