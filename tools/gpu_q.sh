mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "adam or step or compress" 2>&1 | tail -2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
k() { ncu --metrics $M --clock-control none -k regex:"$1" -s 4 -c 2 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/n.csv 2>/dev/null; echo "== $2"; python tools/ncu_csv.py gpurun_out/n.csv | sed 's/bytes_//g'; }
k "k_adam|k_stage2" new
LSP_ADAM_WIDE=0 k "k_adam" adam-old
