# Round-2 capture: C4 launch list + ncu --set full of every step kernel (layer 8).
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_list.err; tail -2 gpurun_out/ncu_list.err
for k in "k_apply_y:apply_y" "k_compress_spmm:compress_spmm" "k_build_y_tile:build_y_tile" "k_stage2_adam:stage2_adam"; do
  re=${k%%:*}; tag=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$re" -s 8 -c 1 -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_$tag.err; tail -1 gpurun_out/ncu_$tag.err
done
ls gpurun_out/prof_*
