# Full GPU check: all parity tests, default bench, compress slot sweep.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err
for pin in "1,2" "1,4" "1,8" "2,2" "2,4"; do
  LSP_COMPRESS_SLOTS="$pin" timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_pin.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_pin.json'));b=d['breakdown'];print('pin=$pin', round(d['ms_per_step'],2), b)"
done
