mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "decompress or compress or step" 2>&1 | tail -3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
prof() { ncu --metrics $M --clock-control none -k regex:"k_apply_y|k_build_y|k_compress" -s 6 -c 6 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/n.csv 2>/dev/null; echo "== $*"; python tools/ncu_csv.py gpurun_out/n.csv | sed 's/bytes_//g'; }
run() { python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$*', 'ms/step',round(d['ms_per_step'],2),'apply',round(b['apply_ms_per_step'],2),'compress',round(b['compress_ms_per_step'],2))" || tail -3 gpurun_out/b.err; }
LSP_APPLY_YB_MB=1000 prof nosub
LSP_APPLY_YB_MB=1000 run nosub
