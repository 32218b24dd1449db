mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_schedule.py -q -x 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print(d['ms_per_step'], d['gpu_launches'], d['config']['cuda_graph'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])" || tail -3 gpurun_out/b.err
