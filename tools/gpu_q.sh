mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "decompress or step or layer" 2>&1 | tail -2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
ncu --metrics $M --clock-control none -k regex:"k_apply_y|k_build_y" -s 4 -c 4 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/n.csv 2>/dev/null; python tools/ncu_csv.py gpurun_out/n.csv | sed 's/bytes_//g'
b() { timeout 600 python bench.py --config $1 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],2),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
b c4 x; b c4-bf16 x
