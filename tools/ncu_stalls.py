"""Summarise an ncu --set full report: key throughput metrics, top stall reasons,
and the share of stall samples per 100-instruction SASS region.
    python tools/ncu_stalls.py report.ncu-rep [--regions]"""
import csv, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
d = dict(zip(h, v))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.avg.per_cycle_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__cycles_elapsed.avg", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_bytes.sum"]
print(d.get("Kernel Name", "")[:100])
for k in keys:
    print(f"  {k} = {d.get(k)} {u[h.index(k)] if k in h else ''}")
st = []
for k, val in zip(h, v):
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try:
            st.append((float(val.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in st) or 1
print("  stalls:", ", ".join(f"{n} {100*x/tot:.0f}%" for x, n in sorted(st, reverse=True)[:8]))
if "--regions" in sys.argv:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hh = rows[1]; data = rows[2:]
    iS = hh.index("Warp Stall Sampling (All Samples)"); iSrc = hh.index("Source")
    s = [int(x[iS]) if x[iS].isdigit() else 0 for x in data]
    t = sum(s) or 1
    for a in range(0, len(data), 100):
        if sum(s[a:a+100]) / t > 0.01:
            print(f"  {a:5d}-{a+100:5d} {100*sum(s[a:a+100])/t:5.1f}%  {data[a][iSrc][:60]}")
    top = sorted(range(len(s)), key=lambda i: -s[i])[:15]
    for i in sorted(top):
        print(f"  {i:5d} {100*s[i]/t:5.1f}%  {data[i][iSrc][:80]}")
