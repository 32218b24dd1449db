# C4 fp32: serial vs pipelined (mode 2) order with the fused stage 2, alternated
mkdir -p gpurun_out
for i in 1 2 3; do for p in 0 2; do
timeout 600 python bench.py --config c4 --pipeline $p --no-e2e --no-cpu-baseline > gpurun_out/pab_$p.json 2>gpurun_out/pab_$p.err
python -c "import json;d=json.load(open('gpurun_out/pab_$p.json'));print('c4 pipeline=$p', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -2 gpurun_out/pab_$p.err
done; done
