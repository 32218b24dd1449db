mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "build_y or layer" 2>&1 | tail -3
b() { timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1 $2', 'ms/step',round(d['ms_per_step'],2),{k:round(v,2) for k,v in b.items() if k.endswith('ms_per_step')})" || tail -3 gpurun_out/b.err; }
LSP_BUILD_Y_TILE=0 b c4 vec
for cb in 48 96 128 192; do LSP_BUILD_Y_TILE=2 LSP_BUILD_Y_CB=$cb b c4 t32cb$cb; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
LSP_BUILD_Y_TILE=2 ncu --metrics $M --clock-control none -k regex:"k_build_y" -s 8 -c 2 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/n.csv 2>/dev/null; python tools/ncu_csv.py gpurun_out/n.csv | sed 's/bytes_//g'
