# bench with the native schedule (default) vs the Python LayerSchedule, graph and eager.
mkdir -p gpurun_out
for v in "--schedule native" "--schedule python" "--schedule native --graph 0" "--schedule python --graph 0"; do
timeout 600 python bench.py $v --no-e2e --no-cpu-baseline > gpurun_out/sb.json 2> gpurun_out/sb.err
python -c "
import json;d=json.load(open('gpurun_out/sb.json'));print('$v', round(d['ms_per_step'],3), d['config']['schedule'], d['gpu_launches'])" || tail -3 gpurun_out/sb.err
done
