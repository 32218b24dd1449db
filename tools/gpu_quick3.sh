# Quick check: Y-build parity tests + C4 / C4-bf16 / C3 bench lines (no e2e / CPU baseline).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -m gpu -x -q -k "build_y or y_build or layer or full" > gpurun_out/pytest_q.log 2>&1; tail -3 gpurun_out/pytest_q.log
for c in c4 c4-bf16 c3; do
timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
python -c "
import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['ms_per_step'],3), d['config'].get('step_hbm_frac_of_measured'), json.dumps({k:round(v,3) for k,v in d['breakdown'].items()}))" || tail -3 gpurun_out/bench_$c.err
done
