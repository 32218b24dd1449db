mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "compress or adam or step" 2>&1 | tail -2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_bytes.sum
k() { ncu --metrics $M --clock-control none -k regex:"$1" -s 2 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/n.csv 2>/dev/null; echo "== $2"; python tools/ncu_csv.py gpurun_out/n.csv | sed 's/bytes_//g' | tail -1; }
LSP_COMPRESS_SPMM=1 k k_compress_spmm spmm
LSP_COMPRESS_SPMM=1 LSP_SPMM_PF=0 k k_compress_spmm spmm-pf0
k k_adam adam
