# Session-5 checks: fused stage-2 + Adam tests (incl. wide d and fallbacks),
# the schedule order per config with the fused kernel, the C5 grid on the final sources.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_adam.py tests/test_bench_contract.py -q > gpurun_out/t3.log 2>&1; tail -2 gpurun_out/t3.log
for c in c4 c4-bf16 c3; do for p in 0 1 2; do
  timeout 600 python bench.py --config $c --pipeline $p --no-e2e --no-cpu-baseline > gpurun_out/pipe_${c}_$p.json 2> gpurun_out/pipe_${c}_$p.err
  python -c "import json;d=json.load(open('gpurun_out/pipe_${c}_$p.json'));print('$c pipeline=$p', round(d['ms_per_step'],3), d['clocks']['reasons'])" || tail -2 gpurun_out/pipe_${c}_$p.err
done; done
timeout 2400 python tools/c5_grid.py gpurun_out/c5_grid.json > gpurun_out/c5_grid.log 2>&1; tail -3 gpurun_out/c5_grid.log
