"""Summarise a gpu_round.sh capture into profiles/<tag>_*.md (tracked).

    python tools/summarize_profiles.py r01 [gpurun_out]

Reads the ncu launch list (gpu__time_duration.sum per launch) and the
`--set full` reports, writes:
  profiles/<tag>_launches.md  per-kernel share of the LAST step in the list
  profiles/<tag>_kernels.md   key metrics of each full capture
  profiles/<tag>_launches.csv the raw per-launch durations (name, grid, block, us)
"""
import csv
import os
import re
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block", "smem/block"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long sb"),
]


def short(name):
    name = re.sub(r"\(.*$", "", name.replace("(anonymous namespace)", "anon"))
    name = re.sub(r"^void ", "", name)
    return name.split("::")[-1]


def launches(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "ns":
            v /= 1000.0
        elif r["Metric Unit"] == "ms":
            v *= 1000.0
        rows.append((short(r["Kernel Name"]), r["Grid Size"], r["Block Size"], v))
    return rows


def last_step(rows):
    # bench with --steps 1 --warmup 1: the step is the final run of launches
    # from the first stage-1 compress of the last step to the end.  Steps
    # start with a compress; find the last index where the layer-0 compress of
    # a step begins (count of stage-1 launches per step = n_layers).
    idx = [i for i, r in enumerate(rows) if r[0].startswith("k_compress_")]
    if not idx:
        return rows
    per_step = len(idx) // 2 if len(idx) % 2 == 0 else len(idx)
    start = idx[len(idx) - per_step]
    return rows[start:]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    got = OrderedDict()
    got["kernel"] = vals[hdr.index("Kernel Name")]
    for key, label in KEYS:
        if key in hdr:
            i = hdr.index(key)
            got[label] = f"{vals[i]} {units[i]}".strip()
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                st[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(vals[i])
            except ValueError:
                pass
    tot = sum(st.values())
    if tot > 0:
        top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
        got["top stalls (pc samples)"] = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top)
    return got


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    os.makedirs("profiles", exist_ok=True)
    rows = launches(os.path.join(src, "launches_c4.csv"))
    with open(f"profiles/{tag}_launches.csv", "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "grid", "block", "us"])
        for r in rows:
            w.writerow([r[0], r[1], r[2], f"{r[3]:.3f}"])
    step = last_step(rows)
    agg = OrderedDict()
    for name, _, _, us in step:
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    total = sum(t for _, t in agg.values())
    with open(f"profiles/{tag}_launches.md", "w") as f:
        f.write(f"# {tag}: ncu launch list, one C4 fp32 step (serialised, cold-cache)\n\n")
        f.write("Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv "
                "python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline`.\n"
                "Per-launch times are serialised and cold-cache; compare SHARES with the "
                "bench's CUDA-event phase split, not absolute times.\n\n")
        f.write("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|\n")
        for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {name} | {n} | {t:.1f} | {t / n:.1f} | {100 * t / total:.1f}% |\n")
        f.write(f"\nTotal kernel time in the step: {total / 1000:.2f} ms over "
                f"{sum(n for n, _ in agg.values())} launches.\n")
    with open(f"profiles/{tag}_kernels.md", "w") as f:
        f.write(f"# {tag}: `ncu --set full` captures (one launch each, layer 8 of the step)\n\n")
        reps = sorted(x[:-8] for x in os.listdir(src) if x.startswith("prof_") and x.endswith(".ncu-rep"))
        for rep in reps:
            p = os.path.join(src, rep + ".ncu-rep")
            if not os.path.exists(p):
                continue
            m = full_metrics(p)
            if not m:
                continue
            f.write(f"## {rep}: `{m.pop('kernel')}`\n\n| metric | value |\n|---|---|\n")
            for k, v in m.items():
                f.write(f"| {k} | {v} |\n")
            f.write("\n")
    sys.path.insert(0, os.getcwd())
    import bench  # the same hash bench.py checks roofline.traffic against

    with open(f"profiles/{tag}_srchash.txt", "w") as f:
        f.write(bench.kernel_source_hash() + "\n")
    print(open(f"profiles/{tag}_launches.md").read())
    print(open(f"profiles/{tag}_kernels.md").read())


if __name__ == "__main__":
    main()
