mkdir -p gpurun_out
./tools/micro/l2_gather.bin > gpurun_out/l2_gather.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_compress_spmm" -s 8 -c 1 -o gpurun_out/prof_spmm python bench.py --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_spmm.err; tail -2 gpurun_out/ncu_spmm.err
cat gpurun_out/l2_gather.txt
