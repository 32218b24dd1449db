# Capture recipe of profiles/r02e_* and r02f_*: all GPU tests, smoke, bench lines for every config,
# C4 ncu launch list + --set full of the step kernels, device-fit timing.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 600 gpurun_out/bench_c4.json; echo
for c in c4-bf16 c3 c2 c4-f64; do
timeout 1500 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
python -c "
import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['ms_per_step'],3), d['config'].get('step_hbm_frac_of_measured'), json.dumps(d.get('fit'))[:300])" || tail -3 gpurun_out/bench_$c.err
done
bash tools/gpu_profile_kernels.sh
timeout 900 python tools/time_fit.py 2048 5504 1024 4 9 > gpurun_out/time_fit.json 2>&1; tail -c 600 gpurun_out/time_fit.json
