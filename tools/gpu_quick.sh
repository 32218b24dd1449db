# Quick GPU check: parity tests matching $1 (pytest -k) and one bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "${1:-compress}" 2>&1 | tail -8
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; python -c "
import json;d=json.load(open('gpurun_out/bench_quick.json'));b=d['breakdown'];print('ms/step',round(d['ms_per_step'],2),'value',round(d['value'],1),{k:round(v,2) for k,v in b.items()})"; tail -3 gpurun_out/bench_quick.err
