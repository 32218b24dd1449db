# Backward-overlap legs (T = 2048, 4096) with the current kernels.
mkdir -p gpurun_out
for T in 2048 4096; do
timeout 900 python bench.py --no-e2e --no-cpu-baseline --overlap-bwd $T --timeline-out gpurun_out/timeline_c4_t$T.json > gpurun_out/ovl$T.json 2> gpurun_out/ovl$T.err
python -c "
import json;d=json.load(open('gpurun_out/ovl$T.json'));print('T=$T', json.dumps(d['overlap']))" || tail -3 gpurun_out/ovl$T.err
done
