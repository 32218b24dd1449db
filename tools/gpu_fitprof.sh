# Launch list (per-kernel time) of a capped device fit at the C3 MLP shape, T targets.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_launches.csv python tools/fitcap.py ${1:-2} ${2:-2048} ${3:-5504} > gpurun_out/fitcap.out 2>&1; tail -2 gpurun_out/fitcap.out
python - <<'PY'
import csv, re, collections
rows=[l for l in open('gpurun_out/fit_launches.csv') if l.startswith('"')]
agg=collections.OrderedDict(); cnt=collections.Counter()
for r in csv.DictReader(rows):
    k=re.sub(r"\(.*","",r["Kernel Name"]).split("::")[-1][:60]
    agg[k]=agg.get(k,0)+float(r["Metric Value"]); cnt[k]+=1
tot=sum(agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1])[:15]: print(f"{k:60s} n={cnt[k]:5d} {v/1e3:9.1f} us  {100*v/tot:5.1f}%")
print("total kernel time us", tot/1e3)
PY
