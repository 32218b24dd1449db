# Apply consumer groups: kNG = 2 (in-tree) vs 1 / 4 (variant libraries).
mkdir -p gpurun_out
run() { for c in c4 c4-bf16; do
timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/ng.json 2> gpurun_out/ng.err
python -c "
import json;d=json.load(open('gpurun_out/ng.json'));b=d['breakdown'];print('$1 $c', round(d['ms_per_step'],3), 'apply', round(b['apply_ms_per_step'],3))" || tail -3 gpurun_out/ng.err
done; }
run ng2
cp paper_2406_10181_b200/liblsp_b200.so /tmp/libng2.so
cp tools/lib_ng1.so paper_2406_10181_b200/liblsp_b200.so; run ng1
cp tools/lib_ng4.so paper_2406_10181_b200/liblsp_b200.so; run ng4
cp /tmp/libng2.so paper_2406_10181_b200/liblsp_b200.so
