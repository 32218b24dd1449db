mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_schedule.py -q -x 2>&1 | tail -2
for dr in "1024 2" "256 4" "1024 4"; do set -- $dr; timeout 300 python bench.py --config c5 --d $1 --r $2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c5 d=$1 r=$2', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))" || echo "c5 $1 $2 failed"; done
