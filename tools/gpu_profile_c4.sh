set -x
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 3000 gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_list.err; tail -3 gpurun_out/ncu_list.err
ncu --set full --clock-control none --import-source on -k regex:k_decompress_band -s 20 -c 2 -o gpurun_out/prof_apply python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_full1.err; tail -3 gpurun_out/ncu_full1.err
ncu --set full --clock-control none --import-source on -k regex:k_compress_stage1 -s 20 -c 2 -o gpurun_out/prof_stage1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_full2.err; tail -3 gpurun_out/ncu_full2.err
ls -la gpurun_out
