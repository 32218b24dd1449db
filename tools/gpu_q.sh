mkdir -p gpurun_out
b() { timeout 300 python bench.py --config $1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $3 > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],3),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
for c in c4 c3; do b $c base ""; b $c side "--side 1"; done
b c4 side-sms100 "--side 1 --sms-compress 120"
b c4 base ""
