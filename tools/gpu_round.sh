# One GPU call: parity tests, bench, launch list, ncu captures of the hot kernels.
set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x 2>&1 | tail -25
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_list.err; tail -3 gpurun_out/ncu_list.err
ncu --set full --clock-control none --import-source on -k regex:k_decompress -s 40 -c 1 -o gpurun_out/prof_apply python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_full1.err; tail -3 gpurun_out/ncu_full1.err
ncu --set full --clock-control none --import-source on -k regex:k_compress_stage1 -s 40 -c 1 -o gpurun_out/prof_stage1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_full2.err; tail -3 gpurun_out/ncu_full2.err
ncu --set full --clock-control none --import-source on -k regex:k_stage2 -s 40 -c 1 -o gpurun_out/prof_stage2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_full3.err; tail -3 gpurun_out/ncu_full3.err
