mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "build_y or y_build" 2>&1 | tail -2
for v in "LSP_BUILD_Y_VEC=1" "LSP_BUILD_Y_VEC=0"; do
env $v timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/yb.json 2> gpurun_out/yb.err; python -c "
import json;d=json.load(open('gpurun_out/yb.json'));b=d['breakdown'];print('$v', 'ms/step',round(d['ms_per_step'],2),'build',round(b['build_y_ms_per_step'],2),'apply',round(b['apply_ms_per_step'],2))" || tail -2 gpurun_out/yb.err
done
