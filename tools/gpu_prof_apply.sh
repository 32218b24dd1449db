# ncu --set full (source) captures of k_apply_y and k_stage2_f4 (layer 8 of a C4 step).
mkdir -p gpurun_out
for k in "k_apply_y:apply_y" "k_stage2:stage2" "k_adam:adam"; do
  re=${k%%:*}; tag=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$re" -s 8 -c 1 -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_$tag.err; tail -1 gpurun_out/ncu_$tag.err
done
