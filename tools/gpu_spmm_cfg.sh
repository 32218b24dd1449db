# Compress stage-1 occupancy experiment: LSP_SPMM_CFG=ctas,u on C4 fp32 / bf16.
mkdir -p gpurun_out
for c in c4 c4-bf16; do
for cfg in 2,8 3,4 2,4 3,8; do
LSP_SPMM_CFG=$cfg timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/spmm_$c_$cfg.json 2> gpurun_out/spmm.err
python -c "
import json;d=json.load(open('gpurun_out/spmm_$c_$cfg.json'));print('$c cfg=$cfg', round(d['ms_per_step'],3), 'compress', round(d['breakdown']['compress_ms_per_step'],3))" || tail -3 gpurun_out/spmm.err
done; done
