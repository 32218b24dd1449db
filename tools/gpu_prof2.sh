# ncu --set full of one launch each of the compress stage-1 and decompress kernels (C4 bench)
mkdir -p gpurun_out
for k in "k_compress_slots:slots" "k_decompress_tma:apply"; do
  re=${k%%:*}; tag=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$re" -s 8 -c 1 -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_$tag.err; tail -3 gpurun_out/ncu_$tag.err
done
