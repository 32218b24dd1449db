mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "compress or layer or full_size or golden" 2>&1 | tail -1
b() { timeout 300 python bench.py --config $1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $3 > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],3),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
b c4 s2v4 ""; b c3 s2v4 ""; b c2 s2v4 ""
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stage2" -s 8 -c 2 --csv python bench.py --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > gpurun_out/n.csv 2>/dev/null; python tools/ncu_csv.py gpurun_out/n.csv
