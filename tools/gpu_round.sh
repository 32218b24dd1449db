# One GPU call: parity tests, bench (all configs), launch list, ncu captures of the hot kernels.
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python bench.py --profile-out gpurun_out/c4_timing_profile.json > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
for cfg in c2 c3 c4-bf16; do timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; cat gpurun_out/bench_$cfg.json | python -c "import json,sys;d=json.load(sys.stdin);print('$cfg', round(d['ms_per_step'],3), 'ms/step', round(d['value'],1), 'GB/s frac', round(d['roofline']['frac'],3), 'step_frac', round(d['config']['step_hbm_frac_of_measured'],3))" || tail -3 gpurun_out/bench_$cfg.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_list.err; tail -2 gpurun_out/ncu_list.err
for k in "k_apply_y:apply_y" "k_compress_spmm:compress_spmm" "k_build_y_vec:build_y" "k_stage2:stage2" "k_adam:adam"; do
  re=${k%%:*}; tag=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$re" -s 8 -c 1 -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_$tag.err; tail -1 gpurun_out/ncu_$tag.err
done
ls gpurun_out
