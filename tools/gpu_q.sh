mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_dp.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --no-e2e --profile-out gpurun_out/c4_timing_profile.json > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print(d['ms_per_step'], d['dp_projection'])" || tail -3 gpurun_out/b.err
