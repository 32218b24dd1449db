# Round-2 bench legs: C4 default line (both CPU baseline modes), backward overlap with a
# timeline, C3 with the fit leg.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 1500 gpurun_out/bench_c4.json; tail -2 gpurun_out/bench_c4.err
for T in ${1:-2048 4096}; do
timeout 900 python bench.py --no-e2e --no-cpu-baseline --overlap-bwd $T --timeline-out gpurun_out/timeline_c4_t$T.json > gpurun_out/bench_c4_ovl$T.json 2> gpurun_out/bench_c4_ovl$T.err; python -c "
import json;d=json.load(open('gpurun_out/bench_c4_ovl$T.json'));print('T=$T', json.dumps(d['overlap']))" || tail -3 gpurun_out/bench_c4_ovl$T.err
done
timeout 1200 python bench.py --config c3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_fit.json 2> gpurun_out/bench_c3_fit.err; python -c "
import json;d=json.load(open('gpurun_out/bench_c3_fit.json'));print('c3', d['ms_per_step'], json.dumps(d.get('fit')))" || tail -3 gpurun_out/bench_c3_fit.err
