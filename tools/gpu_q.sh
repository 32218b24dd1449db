mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "compress or layer or step or golden or conformance" 2>&1 | tail -2
b() { timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],2),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
b c4 s2
b c4-bf16 s2
b c3 s2
b c2 s2
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_stage2" -s 8 -c 2 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/n.csv 2>/dev/null; python tools/ncu_csv.py gpurun_out/n.csv | sed 's/bytes_//g'
