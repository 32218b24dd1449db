# C4 fp32: Y build + apply in L2-sized subgroups (LSP_APPLY_YB_MB) vs the whole layer
mkdir -p gpurun_out
for i in 1 2; do for y in 0 48 96; do
if [ $y = 0 ]; then E=""; else E="LSP_APPLY_YB_MB=$y"; fi
env $E timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline > gpurun_out/yb_$y.json 2>gpurun_out/yb_$y.err
python -c "import json;d=json.load(open('gpurun_out/yb_$y.json'));b=d['breakdown'];print('c4 yb_mb=$y', round(d['ms_per_step'],3), round(b['build_y_ms_per_step'],3), round(b['apply_ms_per_step'],3), d['clocks']['reasons'])" || tail -2 gpurun_out/yb_$y.err
done; done
