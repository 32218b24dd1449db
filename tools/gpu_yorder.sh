# Y-block L2 residency: build order reversed (default) vs forward; sub-grouped build+apply.
mkdir -p gpurun_out
for c in c4 c4-bf16 c3; do
for v in "LSP_BUILD_Y_REVERSE=1" "LSP_BUILD_Y_REVERSE=0" "LSP_APPLY_YB_MB=96" "LSP_APPLY_YB_MB=64"; do
env $v timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/yo.json 2> gpurun_out/yo.err
python -c "
import json;d=json.load(open('gpurun_out/yo.json'));b=d['breakdown'];print('$c $v', round(d['ms_per_step'],3), 'apply', round(b['apply_ms_per_step'],3), 'build', round(b['build_y_ms_per_step'],3))" || tail -3 gpurun_out/yo.err
done; done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_apply_y -s 8 -c 1 python bench.py --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "dram__|gpu__time" 
