# Final verification of a round: GPU tests, smoke, default bench line, the other configs.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; cat gpurun_out/final_c4.json; tail -2 gpurun_out/final_c4.err
for cfg in c2 c3 c4-bf16; do timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline > gpurun_out/final_$cfg.json 2> gpurun_out/final_$cfg.err; python -c "import json;d=json.load(open('gpurun_out/final_$cfg.json'));print('$cfg', round(d['ms_per_step'],3), 'ms/step', round(d['value'],1), 'GB/s frac', round(d['roofline']['frac'],3), 'step_frac', round(d['config']['step_hbm_frac_of_measured'],3))" || tail -3 gpurun_out/final_$cfg.err; done
for dr in "256 4" "1024 2" "1024 4" "1024 8" "4096 4"; do set -- $dr; timeout 300 python bench.py --config c5 --d $1 --r $2 --no-e2e --no-cpu-baseline > gpurun_out/final_c5.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/final_c5.json'));print('c5 d=$1 r=$2', round(d['ms_per_step'],4), 'ms', round(d['value'],1), 'GB/s frac', round(d['roofline']['frac'],3))" || echo "c5 $1 $2 failed"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('reference', d['value'], d['unit'], d['cpu_baseline']['cores'])"
