# C2 (GPT-2 774M, d=512) launch list + ncu --set full of its compress kernels
mkdir -p gpurun_out
B="python bench.py --config c2 --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > /dev/null 2>gpurun_out/ncu_c2.err; tail -1 gpurun_out/ncu_c2.err
for k in "k_compress_spmm:c2_spmm" "k_stage2_adam:c2_s2a"; do
  re=${k%%:*}; tag=${k##*:}
  timeout 600 ncu --set full --clock-control none -k "regex:$re" -s 8 -c 1 -o gpurun_out/prof_$tag $B > /dev/null 2>gpurun_out/ncu_$tag.err; tail -1 gpurun_out/ncu_$tag.err
done
