# C3 bench line with the fit leg (fit allocation fix) + the full C5 d x r grid.
mkdir -p gpurun_out
timeout 1500 python bench.py --config c3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "
import json;d=json.load(open('gpurun_out/bench_c3.json'));print('c3', round(d['ms_per_step'],3), [(p['shape'], round(p['maybe_update_ms'])) for p in d['fit']['per_shape']], d['fit']['amortized_ms_per_step'])" || tail -3 gpurun_out/bench_c3.err
timeout 2400 python tools/c5_grid.py gpurun_out/c5_grid.json > gpurun_out/c5_grid.log 2>&1; tail -3 gpurun_out/c5_grid.log
