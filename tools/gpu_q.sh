mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_compress_spmm" -s 8 -c 1 -o gpurun_out/prof_compress_spmm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_cs.err; tail -1 gpurun_out/ncu_cs.err
