# Compress fixed-slot variants: parity + C4 bench per pinned (CPL,K).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "compress" 2>&1 | tail -5
for pin in "" "1,2" "1,4" "1,8" "2,2" "2,4"; do
  LSP_COMPRESS_SLOTS="$pin" timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_pin.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_pin.json'));b=d['breakdown'];print('pin=$pin', round(d['ms_per_step'],2), 'compress', round(b['compress_ms_per_step'],2))"
done
