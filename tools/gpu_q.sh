mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_dp.py -q -x 2>&1 | tail -3
b() { timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $1 > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1', 'ms/step',round(d['ms_per_step'],2),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
b ""
b "--concurrent 1"
for c in 64 80 96 112; do for u in 0 148; do b "--concurrent 1 --sms-compress $c --sms-update $((u==0 ? 148-c : 148))"; done; done
b "--concurrent 1 --sms-compress 40 --sms-update 108"
b "--concurrent 1 --sms-compress 128 --sms-update 20"
