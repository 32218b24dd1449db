# Block Y build: C4 bench split + ncu capture of one k_build_y launch.
mkdir -p gpurun_out
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python -c "
import json;d=json.load(open('gpurun_out/bench_c4.json'));print('c4', round(d['ms_per_step'],3), json.dumps({k:round(v,3) for k,v in d['breakdown'].items()}))" || tail -3 gpurun_out/bench_c4.err
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_build_y" -s 8 -c 1 -o gpurun_out/prof_yblk python bench.py --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_yblk.err; tail -1 gpurun_out/ncu_yblk.err
