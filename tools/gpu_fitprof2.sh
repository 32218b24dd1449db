# Launch list of a capped device fit (C3 MLP shape, T targets): per-kernel totals and
# per-launch duration classes of the fp64 gather.
mkdir -p gpurun_out
bash tools/gpu_fitprof.sh ${1:-2} ${2:-2048} ${3:-5504}
python - <<'PY'
import csv, re, collections
rows=[l for l in open('gpurun_out/fit_launches.csv') if l.startswith('"')]
h=collections.defaultdict(list)
for r in csv.DictReader(rows):
    k=re.sub(r"\(.*","",r["Kernel Name"]).split("::")[-1][:40]
    h[(k, r["Grid Size"])].append(float(r["Metric Value"]))
for (k,g),v in sorted(h.items(), key=lambda x:-sum(x[1]))[:14]:
    print(f"{k:40s} grid={g:14s} n={len(v):4d} mean={sum(v)/len(v)/1e3:8.1f} us total={sum(v)/1e3:9.1f} us")
PY
