mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json; tail -2 gpurun_out/bench_c4.err
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_compress_spmm" -s 8 -c 1 -o gpurun_out/prof_compress_spmm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_cs.err; tail -1 gpurun_out/ncu_cs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_list.err; tail -2 gpurun_out/ncu_list.err
