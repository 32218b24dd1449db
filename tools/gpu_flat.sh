# Flat-stream gather compress (LSP_SPMM_FLAT=1): parity, then compress time per config vs the padded form.
mkdir -p gpurun_out/flat
LSP_SPMM_FLAT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "compress_paths or determinism or full_size or value_refresh" 2>&1 | tail -3
for c in c4 c4-bf16 c3 c2; do for v in 0 1; do
LSP_SPMM_FLAT=$v timeout 600 python bench.py --config $c --fit-every 0 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/flat/$c-$v.json 2>gpurun_out/flat/$c-$v.err
python -c "
import json;d=json.load(open('gpurun_out/flat/$c-$v.json'));print('$c flat=$v', round(d['ms_per_step'],3), round(d['breakdown']['compress_ms_per_step'],3))" || tail -3 gpurun_out/flat/$c-$v.err
done; done
