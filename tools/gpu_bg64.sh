# Gather-compress items of 64 bins (tools/lib_bg64.so) vs 32 (in-tree) on the small-m configs.
mkdir -p gpurun_out
run() { for c in c3 c2 c4-bf16 c4; do
timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/bg.json 2> gpurun_out/bg.err
python -c "
import json;d=json.load(open('gpurun_out/bg.json'));b=d['breakdown'];print('$1 $c', round(d['ms_per_step'],3), 'compress', round(b['compress_ms_per_step'],3))" || tail -3 gpurun_out/bg.err
done; }
run bg32
cp paper_2406_10181_b200/liblsp_b200.so /tmp/lib32.so; cp tools/lib_bg64.so paper_2406_10181_b200/liblsp_b200.so
run bg64
cp /tmp/lib32.so paper_2406_10181_b200/liblsp_b200.so
