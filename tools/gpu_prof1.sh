# ncu --set full of one launch of the kernel matching regex $1 (C4 bench, layer 8)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$1" -s 8 -c 1 -o gpurun_out/prof_$2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_$2.err; tail -3 gpurun_out/ncu_$2.err
