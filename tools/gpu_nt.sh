# A/B runs: fused-stage-2 tests, then C2 / C4 / C3 bench lines (phase split)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused_adam.py -q 2>&1 | tail -1
for c in c2 c4 c3; do
timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/nt_$c.json 2>gpurun_out/nt_$c.err
python -c "import json;d=json.load(open('gpurun_out/nt_$c.json'));print('$c', round(d['ms_per_step'],3), {k[:-12]:round(v,3) for k,v in d['breakdown'].items() if k.endswith('ms_per_step')}, d['clocks']['reasons'])" || tail -2 gpurun_out/nt_$c.err
done
