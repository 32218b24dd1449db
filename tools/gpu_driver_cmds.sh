# The driver's round-end commands at N=1 (both arms), timed.
mkdir -p gpurun_out
t0=$(date +%s); timeout 1200 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_ours.json 2> gpurun_out/drv_ours.err; echo "ours wall $(( $(date +%s) - t0 )) s"; tail -1 gpurun_out/drv_ours.err
t0=$(date +%s); timeout 1200 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_ref.json 2> gpurun_out/drv_ref.err; echo "ref wall $(( $(date +%s) - t0 )) s"; tail -1 gpurun_out/drv_ref.err
python3 -c "
import json
a=json.load(open('gpurun_out/drv_ours.json')); b=json.load(open('gpurun_out/drv_ref.json'))
print('ours', a['ms_per_step'], a['value'], a['e2e']['value'], a['roofline']['frac'], a['roofline']['traffic_stale'], a['clocks'])
print('ref', b['ms_per_step'], b['value'], b['e2e']['value'])"
