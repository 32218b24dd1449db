# C4 in the reference's own precision (fp64 G, W, projectors, state).
mkdir -p gpurun_out
timeout 1200 python bench.py --config c4-f64 > gpurun_out/bench_c4-f64.json 2> gpurun_out/bench_c4-f64.err
python -c "
import json;d=json.load(open('gpurun_out/bench_c4-f64.json'));print('c4-f64', round(d['ms_per_step'],3), round(d['value'],1), d['config']['step_hbm_frac_of_measured'], d['roofline']['frac'], d['breakdown'], d['e2e'], d['cpu_baseline']['value'], d['gpu_launches'])" || tail -20 gpurun_out/bench_c4-f64.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4-f64.csv python bench.py --config c4-f64 --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_f64.err; tail -2 gpurun_out/ncu_f64.err
python - <<'PY'
import csv, re, collections
rows = [l for l in open("gpurun_out/launches_c4-f64.csv") if l.startswith('"')]
agg = collections.OrderedDict()
for r in csv.DictReader(rows):
    k = re.sub(r"\(.*", "", r["Kernel Name"]).split("::")[-1]
    a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += float(r["Metric Value"].replace(",", "")) / (1e3 if r["Metric Unit"] == "nsecond" else 1)
tot = sum(v[1] for v in agg.values())
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} {n:4d} {us:10.1f} us {us/n:8.1f} {100*us/tot:5.1f}%")
PY
