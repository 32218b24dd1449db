# One ncu --set full capture of kernel regex $1 (bench config $2, default c4), layer 8 of the step.
mkdir -p gpurun_out
tag=${3:-k}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s 8 -c 1 -o gpurun_out/prof_$tag python bench.py --config ${2:-c4} --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_$tag.err; tail -2 gpurun_out/ncu_$tag.err
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_$tag.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page details --csv > gpurun_out/prof_$tag.details.csv 2>/dev/null
ls -la gpurun_out/prof_$tag*
