# Quick GPU check: parity tests matching $1 (pytest -k) and one C4 bench line with its breakdown.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "${1:-build_y}" 2>&1 | tail -4
for cfg in ${2:-c4}; do
timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$cfg.json'));b=d['breakdown'];print('$cfg', 'ms/step',round(d['ms_per_step'],2),'value',round(d['value'],1),'frac',round(d['config']['step_hbm_frac_of_measured'],3),{k:round(v,2) for k,v in b.items()})" || tail -3 gpurun_out/bench_$cfg.err
done
