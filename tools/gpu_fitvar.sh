# Fit time variance: trial counts (LSP_FIT_TRACE) and SM clocks during C3-shape maybe_updates.
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 500 > gpurun_out/fit_smi.csv &
SMI=$!
LSP_FIT_TRACE=1 timeout 600 python tools/time_fit_c3.py 2>&1 | tail -14
kill $SMI
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/fit_smi.csv')))[1:]
mhz=[int(r[1].split()[0]) for r in rows if len(r)>3]
print('sm MHz min/median/max', min(mhz), sorted(mhz)[len(mhz)//2], max(mhz), 'reasons', sorted(set(r[3].strip() for r in rows if len(r)>3)))
PY
