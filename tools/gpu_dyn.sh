# Dynamic heaviest-first stage-1 schedule: every GPU test, then A/B bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_dyn.log 2>&1; tail -2 gpurun_out/pytest_dyn.log
for c in c2 c4 c3 c4-bf16; do for D in 1 0; do
LSP_SPMM_DYN=$D timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/dyn_${c}_$D.json 2>gpurun_out/dyn_${c}_$D.err
python -c "import json;d=json.load(open('gpurun_out/dyn_${c}_$D.json'));print('$c dyn=$D', round(d['ms_per_step'],3), {k[:-12]:round(v,3) for k,v in d['breakdown'].items() if k.endswith('ms_per_step')}, d['clocks']['reasons'])" || tail -2 gpurun_out/dyn_${c}_$D.err
done; done
