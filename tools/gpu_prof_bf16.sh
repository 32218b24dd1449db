# ncu --set full of the bf16 gather compress (C4-bf16, layer 8).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_compress_spmm" -s 8 -c 1 -o gpurun_out/prof_spmm_bf16 python bench.py --config c4-bf16 --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_bf16.err; tail -1 gpurun_out/ncu_bf16.err
