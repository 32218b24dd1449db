# C5: r/d sweep on one 4096 x 11008 fp32 matrix (BASELINE configs[4], "r" and "d"
# in the reference's naming: d = subspace width, r = nonzeros per row)
mkdir -p gpurun_out
for d in 256 512 1024 2048 4096; do for r in 2 4 8; do
  timeout 300 python bench.py --config c5 --d $d --r $r --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5.json 2> gpurun_out/c5.err
  python -c "
import json;x=json.load(open('gpurun_out/c5.json'));b=x['breakdown']
print('d=$d r=$r', 'ms',round(x['ms_per_step'],3),'GB/s',round(x['value'],1),'step_frac',round(x['config']['step_hbm_frac_of_measured'],3),'apply_frac',round(x['roofline']['frac'],3),{k[:-12]:round(v,3) for k,v in b.items() if k.endswith('ms_per_step')})" 2>/dev/null || (echo "d=$d r=$r FAILED"; tail -2 gpurun_out/c5.err)
done; done
