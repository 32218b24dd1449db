# Full validation: every GPU test, smoke, the default bench line (N=1) and the reference arm.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; python -c "
import json;d=json.load(open('gpurun_out/bench_c4.json'));print('c4', round(d['ms_per_step'],3), round(d['value'],1), d['config']['schedule'], d['roofline']['frac'], d['roofline']['traffic_stale'], d['e2e']['value'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])" || tail -3 gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -c 400 gpurun_out/ref.json
