mkdir -p gpurun_out
timeout 900 python tools/dbg_r2.py "515,700,96,2;3,64,32,2"
timeout 1500 python -m pytest tests -q -m gpu --timeout 240 2>&1 | tail -3
