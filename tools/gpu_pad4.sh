# Padding unit of the gather-compress CSC table: 8 (default) vs 4 (tools/lib_pad4.so).
mkdir -p gpurun_out
run() { for c in c2 c3 c4 c4-bf16; do
timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/p4.json 2> gpurun_out/p4.err
python -c "
import json;d=json.load(open('gpurun_out/p4.json'));b=d['breakdown'];print('$1 $c', round(d['ms_per_step'],3), 'compress', round(b['compress_ms_per_step'],3))" || tail -3 gpurun_out/p4.err
done; }
run pad8
cp paper_2406_10181_b200/liblsp_b200.so /tmp/lib8.so; cp tools/lib_pad4.so paper_2406_10181_b200/liblsp_b200.so
run pad4
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "compress" 2>&1 | tail -1
cp /tmp/lib8.so paper_2406_10181_b200/liblsp_b200.so
