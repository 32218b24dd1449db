# Launch list (per-kernel time) of a capped device fit at the C3 MLP shape, T targets.
mkdir -p gpurun_out
cat > /tmp/fitcap.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2406_10181_b200 as lsp
m, n, d, r, T = int(sys.argv[2]) if len(sys.argv) > 2 else 2048, int(sys.argv[3]) if len(sys.argv) > 3 else 5504, 1024, 4, int(sys.argv[1])
P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(1, 0x1A171, 2))
Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(1, 0x1A171, 3))
pair = lsp.DevicePair(P, Q)
tg = [torch.randn(m, n, device="cuda") for _ in range(T)]
rep = pair.fit(tg, lsp.FitConfig(max_steps=5, timeout_steps=5))
torch.cuda.synchronize()
print("steps", rep.steps)
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_launches.csv python /tmp/fitcap.py ${1:-2} ${2:-2048} ${3:-5504} > gpurun_out/fitcap.out 2>&1; tail -2 gpurun_out/fitcap.out
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
