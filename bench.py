#!/usr/bin/env python
"""Benchmark of the LSP projector hot path (BASELINE.json metric):

    grad GB/s (compress + decompress + apply) vs HBM peak; ms/step per layer stack

A step = one pass of the hot path over one synthetic gradient per linear layer
of the model: per matrix, compress S = P^T G Q, (all-reduce S over ranks),
subspace Adam, fused decompress-and-apply W -= lr P dS Q^T, layers visited in
backward order.  Inputs are resident in HBM (larger than L2: no flush needed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

Under torchrun (N > 1) every rank processes its own synthetic gradients (weak
scaling, data parallel); the per-matrix S is all-reduced (mean) over NCCL and the
update is replicated.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KINIT = 0x1A171  # proj/src/trainer.cpp:23 (projector init tag)

# name -> (description, layers, [(m, n, count)], d (subspace), r (nnz/row), g dtype, w dtype)
CONFIGS = {
    "c1": ("single 1024x1024 weight, d=256, r=4 (BASELINE configs[0])", 1,
           [(1024, 1024, 1)], 256, 4, "f32", "f32"),
    "c2": ("GPT-2 774M 36-layer stack, d=512, r=4, fp32 (BASELINE configs[1])", 36,
           [(1280, 1280, 4), (1280, 5120, 1), (5120, 1280, 1)], 512, 4, "f32", "f32"),
    "c3": ("1.3B decoder 24-layer stack, d=1024, r=4, bf16 (BASELINE configs[2])", 24,
           [(2048, 2048, 4), (2048, 5504, 2), (5504, 2048, 1)], 1024, 4, "bf16", "bf16"),
    "c4": ("Llama-7B 32-layer stack, d=1024, r=4, fp32 (BASELINE configs[3])", 32,
           [(4096, 4096, 4), (4096, 11008, 2), (11008, 4096, 1)], 1024, 4, "f32", "f32"),
    "c4-bf16": ("Llama-7B 32-layer stack, d=1024, r=4, bf16 (BASELINE configs[3])", 32,
                [(4096, 4096, 4), (4096, 11008, 2), (11008, 4096, 1)], 1024, 4, "bf16", "bf16"),
    # the reference's own precision: fp64 G, W, projectors, S/M/V (not a BASELINE
    # config; the device path is bit-exact to the reference's Adam in fp64)
    "c4-f64": ("Llama-7B 32-layer stack, d=1024, r=4, fp64 (the reference's precision)", 32,
               [(4096, 4096, 4), (4096, 11008, 2), (11008, 4096, 1)], 1024, 4, "f64", "f64"),
}
BYTES = {"f32": 4, "bf16": 2, "f64": 8}


def dtype_label(gdt, wdt):
    """Arithmetic type of the step's big streams (G read, W read-modify-write);
    S/M/V and every accumulation are fp32 (fp64 for the f64 config)."""
    return gdt if gdt == wdt else f"g={gdt},w={wdt}"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS) + ["c5"])
    ap.add_argument("--d", type=int, default=None, help="c5 sweep: subspace width")
    ap.add_argument("--r", type=int, default=None, help="c5 sweep: nonzeros per row")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--profile-out", default=None,
                    help="write the measured per-layer times as a reference TimingProfile JSON "
                         "(paper_2406_10181_b200/calibrate.py) for --profile-world ranks")
    ap.add_argument("--profile-world", type=int, default=8)
    ap.add_argument("--busbw-gbs", type=float, default=700.0,
                    help="all-reduce bus bandwidth for --profile-out (nominal NVLink 5 figure; "
                         "not measured on one GPU)")
    ap.add_argument("--graph", type=int, default=1,
                    help="1 (default): capture one step in a CUDA graph and replay it in the "
                         "timed region (N=1 only; the per-phase split comes from one eager "
                         "step just before); 0: eager launches")
    ap.add_argument("--schedule", choices=("native", "python"), default="native",
                    help="step driver of the timed region: the library's C++ schedule "
                         "(lsp_schedule_step, default) or schedule.LayerSchedule (Python); "
                         "the per-phase split always uses LayerSchedule's hooks")
    ap.add_argument("--pipeline", type=int, default=-1,
                    help="1: stage 2 + Adam of layer l on a side stream beside the Y build of "
                         "layer l+1 (apply alone); 2: also beside its apply; 0: serial; "
                         "-1 (default): 2 for bf16 W (measured faster: C3 5.77 -> 5.53 ms, "
                         "C4-bf16 18.43 -> 18.24), 0 for fp32 W (C4 24.51 vs 24.68)")
    ap.add_argument("--concurrent", type=int, default=0,
                    help="1: compress and update chains on two streams (schedule.py)")
    ap.add_argument("--partition", type=int, default=0,
                    help="SMs of the green-context partition running every layer's compress "
                         "stage 1 while the rest run stage 2 / Adam / Y build / apply "
                         "(lsp_schedule_set_partition; native schedule only); 0: off")
    ap.add_argument("--sms-compress", type=int, default=0, help="lsp_set_sm_budget compress SMs")
    ap.add_argument("--sms-update", type=int, default=0, help="lsp_set_sm_budget update SMs")
    ap.add_argument("--overlap-bwd", type=int, default=0, metavar="TOKENS",
                    help="backward-overlap mode: stand-in weight-gradient GEMMs G = X^T dY "
                         "(TOKENS rows) on the compute stream produce every G, the LSP chain "
                         "runs on a side stream gated per layer (schedule.py); reports the "
                         "exposed LSP time vs backward alone (0: off)")
    ap.add_argument("--bwd-carveout", type=int, default=0,
                    help="with --overlap-bwd: SMs the backward GEMMs leave free "
                         "(torch SM carve-out for cuBLAS) and the LSP persistent grids use "
                         "(lsp_set_sm_budget); 0: no partition")
    ap.add_argument("--lsp-priority", type=int, default=0,
                    help="with --overlap-bwd: 1 = the LSP stream gets the higher priority")
    ap.add_argument("--timeline-out", default=None,
                    help="with --overlap-bwd: write the per-stream phase timeline of one step")
    ap.add_argument("--fit-every", type=int, default=None,
                    help="projector refresh cadence (trainer check_freq); default 100 for c3 "
                         "(BASELINE configs[2]), 0 elsewhere: times maybe_update per shape")
    ap.add_argument("--fit-ring", type=int, default=8,
                    help="extra ring gradients passed to the fit (trainer ring_capacity)")
    ap.add_argument("--c5-layers", type=int, default=4,
                    help="c5: independent 4096 x 11008 matrices per step (inputs > L2)")
    return ap.parse_args()


def workload(args):
    if args.config == "c5":
        d, r = args.d or 1024, args.r or 4
        return (f"4096x11008 d/r sweep, d={d}, r={r}, fp32 (BASELINE configs[4])",
                args.c5_layers, [(4096, 11008, 1)], d, r, "f32", "f32")
    desc, L, shapes, d, r, gdt, wdt = CONFIGS[args.config]
    if args.d:
        d = args.d
    if args.r:
        r = args.r
    return desc, L, shapes, d, r, gdt, wdt


def matrices(L, shapes):
    """Per-layer matrix list in the reference's (fan_in x fan_out) orientation."""
    out = []
    for layer in range(L):
        for (m, n, cnt) in shapes:
            for _ in range(cnt):
                out.append((layer, m, n))
    return out


def b_alg(m, n, d, r, bg, bw, bv=4):
    """algorithmic HBM bytes of one matrix step (bv = bytes of the
    compute type: projector values and the S, M, V, delta state, 24 d^2 in fp32)."""
    return m * n * (bg + 2 * bw) + 6 * bv * d * d + 2 * (m + n) * r * (4 + bv)


def apply_bytes(m, n, d, r, bw, bv=4):
    """Algorithmic bytes of one decompress-and-apply launch: W read+write once,
    delta^T read once, CSR (pos, val) of P and Q read once."""
    return 2 * m * n * bw + bv * d * d + (m + n) * r * (4 + bv)


def compress_bytes(m, n, d, r, bg, bv=4):
    """Algorithmic bytes of one compress (stage 1 + 2): G read once, S written once,
    projector entries read once."""
    return m * n * bg + bv * d * d + (m + n) * r * (4 + bv)


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


KERNEL_SOURCES = ("apply.cu", "compress.cu", "compress_spmm.cu", "elementwise.cu", "layer.cu",
                  "core.cuh", "tma.cuh", "adam_math.cuh")


def kernel_source_hash():
    """sha256 over the step kernels' sources: a committed ncu capture is current
    only if it was taken with the same sources (profiles/<tag>_srchash.txt)."""
    import hashlib

    h = hashlib.sha256()
    for f in KERNEL_SOURCES:
        p = os.path.join(ROOT, "paper_2406_10181_b200", "csrc", f)
        if os.path.exists(p):
            h.update(open(p, "rb").read())
    return h.hexdigest()


def profiled_traffic(kernel_prefix, config):
    """DRAM bytes (read + write) of one launch of the roofline kernel from the
    committed ncu --set full summary (profiles/<round>_kernels.md, captured with
    this bench's own C4 command); None for other configs or when absent.
    Returns (bytes, source, stale): stale when the capture's source hash
    (profiles/<tag>_srchash.txt) differs from the current kernel sources."""
    if config != "c4":
        return None, None, None
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_kernels.md")))
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in reversed(files):
        text = open(path).read()
        for sec in text.split("## ")[1:]:
            head = sec.splitlines()[0]
            if kernel_prefix not in head:
                continue
            vals = {}
            for key in ("dram read", "dram write"):
                m = re.search(r"\| %s \| ([0-9.]+) (\w+) \|" % key, sec)
                if m:
                    vals[key] = float(m.group(1)) * units.get(m.group(2), 1)
            if len(vals) == 2:
                hp = path.replace("_kernels.md", "_srchash.txt")
                cap = open(hp).read().strip() if os.path.exists(hp) else None
                return (vals["dram read"] + vals["dram write"], os.path.relpath(path, ROOT),
                        cap != kernel_source_hash())
    return None, None, None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# CPU baseline: the reference (oracle/_ref) or the oracle port, on host cores
# ---------------------------------------------------------------------------
def cpu_info():
    """nproc and the CPU model (lscpu, else /proc/cpuinfo)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    if model is None:
        try:
            for line in open("/proc/cpuinfo"):
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        except OSError:
            pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model}


def cpu_baseline(desc, L, shapes, d, r, gdt, lr, reps=1, single=True):
    """The reference's own step (oracle/_ref: compress, adam_step, W -= decompress*lr)
    timed on the host cores in two modes: all cores (std::threads
    over independent matrices, a bounded sample of layers) -> "value"; and one
    thread, one matrix of each layer shape, serial -> "single_thread"."""
    import oracle

    kind = "reference" if oracle.available("reference") else "port"
    O = oracle.Oracle(kind)
    info = cpu_info()
    cores = info["nproc"]
    per_layer = sum(c for _, _, c in shapes)
    layers = max(1, cores // per_layer)
    rng = np.random.default_rng(0)
    jobs = []
    for (m, n, cnt) in shapes:
        P = O.init_sparse(m, d, r, O.derive_seed(1, KINIT, 0))
        Q = O.init_sparse(n, d, r, O.derive_seed(1, KINIT, 1))
        g = rng.standard_normal((m, n)).astype(np.float32).astype(np.float64)
        w = (0.02 * rng.standard_normal((m, n))).astype(np.float32).astype(np.float64)
        jobs.append((P, Q, g, w, cnt * layers))
    if kind != "reference":
        # the port has no threaded timer: time one matrix per shape serially
        t0 = time.perf_counter()
        for P, Q, g, w, cnt in jobs:
            s = O.compress(P, Q, g)
            z = np.zeros_like(s)
            _, _, de, _ = O.adam_step(z, z, s, 0)
            O.decompress_apply(P, Q, de, lr, w)
        t = time.perf_counter() - t0
        gb = sum(P.n_rows * Q.n_rows for P, Q, *_ in jobs) * BYTES[gdt] / 1e9
        return {"value": gb / t, "unit": "GB/s", "cores": 1, "kind": kind, **info,
                "sample": f"one matrix of each layer shape, serial, {t:.1f}s"}, t
    threads = sum(j[4] for j in jobs)
    times = []
    for _ in range(reps):
        res = [0.0] * len(jobs)

        def run(i, job):
            P, Q, g, w, cnt = job
            res[i] = O.time_step(P, Q, g, w, lr, cnt, cnt)

        th = [threading.Thread(target=run, args=(i, j)) for i, j in enumerate(jobs)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        times.append(time.perf_counter() - t0)
    t = float(np.median(times))
    gb = layers * sum(m * n * c for m, n, c in shapes) * BYTES[gdt] / 1e9
    out = {"value": gb / t, "unit": "GB/s", "cores": threads, "kind": kind, **info,
           "sample": (f"{layers} layer(s) = {threads} matrices of the {desc.split(',')[0]} "
                      f"shapes, one reference step each (compress, adam_step, "
                      f"W -= decompress*lr) on {threads} std::threads, median of {reps}; "
                      f"{t:.1f}s per sample")}
    if single:
        ts = [O.time_step(P, Q, g, w, lr, 1, 1) for P, Q, g, w, _ in jobs]
        gb1 = sum(P.n_rows * Q.n_rows for P, Q, *_ in jobs) * BYTES[gdt] / 1e9
        out["single_thread"] = {
            "value": gb1 / sum(ts), "unit": "GB/s", "cores": 1,
            "sample": ("one matrix of each layer shape (" +
                       ", ".join(f"{P.n_rows}x{Q.n_rows}: {x:.2f}s" for (P, Q, *_), x in
                                 zip(jobs, ts)) + "), one reference step each, 1 thread")}
    return out, t


def run_reference(args):
    desc, L, shapes, d, r, gdt, wdt = workload(args)
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    samples = []
    nrun = args.warmup + args.steps
    for i in range(nrun):
        cb, t = cpu_baseline(desc, L, shapes, d, r, gdt, args.lr, single=(i == nrun - 1))
        samples.append(cb)
    vals = [c["value"] for c in samples[args.warmup:]]
    v = float(np.median(vals))
    cb = dict(samples[-1])
    cb["value"] = v
    total_gb = L * sum(m * n * c for m, n, c in shapes) * BYTES[gdt] / 1e9
    line = {"metric": "grad GB/s (compress+decompress+apply)", "value": v, "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total_gb / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "d": d, "r": r, "layers": L,
                       "note": "ms_per_step extrapolated from the bounded sample to the full stack"},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2406_10181_b200 as lsp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    desc, L, shapes, d, r, gdt, wdt = workload(args)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f64": torch.float64}
    compute = "f64" if gdt == "f64" else "f32"
    mats = matrices(L, shapes)

    # ---- setup (not timed): one lsp.Layer (grouped launches) per model layer ----
    items, layers = [], []
    gen = torch.Generator(device=dev)
    for layer_idx in range(L):
        pairs = []
        for idx, (lay, m, n) in enumerate(mats):
            if lay != layer_idx:
                continue
            # projectors: the reference trainer seed path, identical on every rank
            pp, pv = lsp.init_sparse(m, d, r, lsp.derive_seed(args.seed, KINIT, 2 * idx))
            qp, qv = lsp.init_sparse(n, d, r, lsp.derive_seed(args.seed, KINIT, 2 * idx + 1))
            pair = lsp.DevicePair(lsp.DeviceProjector(m, d, r, pp, pv, compute),
                                  lsp.DeviceProjector(n, d, r, qp, qv, compute))
            gen.manual_seed(lsp.derive_seed(args.seed, 0x6, idx * world + rank))
            g = torch.randn(m, n, device=dev, generator=gen).to(tdt[gdt])
            w = (0.02 * torch.randn(m, n, device=dev, generator=gen)).to(tdt[wdt])
            items.append(dict(m=m, n=n, pair=pair, g=g, w=w))
            pairs.append((pair, g, w))
        lay = lsp.Layer([p for p, _, _ in pairs])
        for i, (_, g, w) in enumerate(pairs):
            lay.bind(i, g, w)
        layers.append(lay)
    torch.cuda.synchronize()
    order = list(reversed(range(L)))  # backward order: last layer's gradients arrive first

    stream = torch.cuda.current_stream()
    from paper_2406_10181_b200.schedule import LayerSchedule

    ev = {(ph, li): (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for ph in ("compress", "adam", "build", "apply") for li in range(L)}
    recording = [False]

    def record(ph, li, when):
        if recording[0]:
            ev[(ph, li)][0 if when == "begin" else 1].record(torch.cuda.current_stream())

    # compress(l) -> all-reduce(S_l) async -> finish(l+1): the all-reduce of layer l
    # overlaps the compress of layer l-1 (paper_2406_10181_b200/schedule.py)
    lsp.set_sm_budget(args.sms_compress, args.sms_update)
    streams = None
    if args.concurrent:
        streams = (torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
    # N > 1: the library's own NCCL communicator carries the S all-reduce
    # (lsp_layer_allreduce on a comm stream; torch.distributed only bootstraps
    # the id and runs the barriers / max-over-ranks timing)
    comm = lsp.Comm.from_group() if world > 1 else None
    pipeline = args.pipeline if args.pipeline >= 0 else (2 if wdt == "bf16" else 0)
    if streams is not None:
        pipeline = 0
    sched = LayerSchedule(layers, args.lr, comm=comm, record=record, streams=streams)
    native = None
    if args.schedule == "native" and streams is None:
        # csrc/schedule.cpp: the same step as LayerSchedule (bitwise), with the
        # pipelined order when selected
        native = lsp.Schedule(layers, comm=comm, pipeline=0 if args.partition else pipeline,
                              partition=args.partition)
    elif pipeline:
        sched = LayerSchedule(layers, args.lr, comm=comm, record=record, pipeline=pipeline)

    def one_step(record=False):
        recording[0] = record
        if native is not None and not record:
            native.step(args.lr)
        else:
            sched.step()
        recording[0] = False

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    graph, graph_launches = None, 0
    if args.graph:  # the NCCL all-reduce on the comm stream is captured too (N > 1)
        one_step(record=True)  # per-phase split (eager), outside the timed region
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        g0 = lsp.launch_count()
        with torch.cuda.graph(graph):
            one_step()
        graph_launches = lsp.launch_count() - g0
        graph.replay()  # warm the graph once
        torch.cuda.synchronize()

    # ---- timed region -------------------------------------------------------
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lsp.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            one_step(record=(k == args.steps - 1))
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = lsp.launch_count() - launches0 + graph_launches * (args.steps if graph else 0)
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / args.steps
    comp_ms = [ev[("compress", li)][0].elapsed_time(ev[("compress", li)][1]) for li in range(L)]
    adam_ms = [ev[("adam", li)][0].elapsed_time(ev[("adam", li)][1]) for li in range(L)]
    app_ms = [ev[("apply", li)][0].elapsed_time(ev[("apply", li)][1]) for li in range(L)]
    try:
        build_ms = [ev[("build", li)][0].elapsed_time(ev[("build", li)][1]) for li in range(L)]
    except RuntimeError:  # layer without a split apply
        build_ms = [0.0] * L
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    for lay in layers:
        lay.check()  # no non-finite gradients were seen

    bg, bw = BYTES[gdt], BYTES[wdt]
    grad_bytes = sum(it["m"] * it["n"] for it in items) * bg
    value = world * grad_bytes / (ms * 1e-3) / 1e9
    bv = BYTES[compute]
    balg = sum(b_alg(it["m"], it["n"], d, r, bg, bw, bv) for it in items)
    peak, peak_src = measured_peaks()
    # dominant kernel: the grouped decompress-and-apply (one k_decompress_band
    # launch per layer, bracketed alone by the "apply" events)
    app_bytes = sum(apply_bytes(it["m"], it["n"], d, r, bw, bv) for it in items) / L
    comp_bytes = sum(compress_bytes(it["m"], it["n"], d, r, bg, bv) for it in items) / L
    app_avg = float(np.mean(app_ms))
    comp_avg = float(np.mean(comp_ms))
    app_ach = app_bytes / (app_avg * 1e-3) / 1e9
    traffic, traffic_src, traffic_stale = profiled_traffic("k_apply_y<float", args.config)
    comp_ach = comp_bytes / (comp_avg * 1e-3) / 1e9
    tsum = sum(app_ms) + sum(comp_ms) + sum(adam_ms) + sum(build_ms)
    line = {
        "metric": "grad GB/s (compress+decompress+apply)",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dtype_label(gdt, wdt),
        "data": "synthetic (torch.randn gradients/weights in HBM; projectors from the reference "
                "trainer seed path)",
        "config": {"workload": desc, "matrices": len(items), "layers": L, "d": d, "r": r,
                   "g_dtype": gdt, "w_dtype": wdt,
                   "params": int(sum(it["m"] * it["n"] for it in items)),
                   "l2": "inputs larger than L2 (%.1f GB of G per rank, streamed once)"
                         % (grad_bytes / 1e9),
                   "parallelism": f"dp{world}",
                   "cuda_graph": (("one captured step replayed per timed step; phase split "
                                   "and roofline launch times from one eager step before it")
                                  if graph is not None else False),
                   "streams": ("2 (compress | update, SM budget %d | %d)"
                               % (args.sms_compress, args.sms_update)) if args.concurrent else "1",
                   "schedule": ("native (lsp_schedule_step, csrc/schedule.cpp)" if native is not None
                                else "python (schedule.LayerSchedule)"),
                   "pipeline": pipeline,
                   "partition_sms": (list(native.partition) if native is not None and args.partition
                                     else None),
                   "step_hbm_bytes_alg": balg,
                   "step_hbm_frac_of_measured": balg / (ms * 1e-3) / 1e9 / peak,
                   "step_hbm_frac_of_8TBs": balg / (ms * 1e-3) / 1e9 / 8000.0},
        "roofline": {"kernel": ("k_apply_y (grouped streaming decompress-and-apply W -= lr P Y, "
                                "1 launch per layer; Y = delta Q^T built by k_build_y_tile just "
                                "before, timed separately as build_ms)") if compute == "f32" else
                               ("k_decompress_tma (grouped fp64 decompress-and-apply, Y band "
                                "built in-kernel from delta^T, 1 launch per layer)"),
                     "bound": "hbm", "achieved": app_ach, "peak": peak, "unit": "GB/s",
                     "frac": app_ach / peak, "traffic": traffic,
                     "traffic_source": (f"{traffic_src}: ncu --set full dram__bytes_read.sum + "
                                        "dram__bytes_write.sum of one launch (includes the "
                                        "Y-block reads from HBM)") if traffic else None,
                     "traffic_stale": traffic_stale,
                     "peak_source": peak_src,
                     "bytes_per_launch_avg": app_bytes, "avg_launch_ms": app_avg,
                     "share_of_step": sum(app_ms) / (ms if ms > 0 else 1)},
        "breakdown": {"compress_ms_per_step": sum(comp_ms), "adam_ms_per_step": sum(adam_ms),
                      "build_y_ms_per_step": sum(build_ms),
                      "apply_ms_per_step": sum(app_ms), "other_ms_per_step": ms - tsum,
                      "compress_achieved_gbs": comp_ach, "compress_frac": comp_ach / peak,
                      "apply_achieved_gbs": app_ach},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if args.profile_out and rank == 0:
        from paper_2406_10181_b200 import calibrate as cal

        per_layer = len(items) // L
        prof = cal.b200_profile([c * 1e-3 for c in comp_ms],
                                [(a + b + c) * 1e-3 for a, b, c in zip(adam_ms, build_ms, app_ms)],
                                [per_layer * d * d * 4.0] * L, args.profile_world,
                                args.busbw_gbs * 1e9, d=d)
        cal.save_profile(prof, args.profile_out)
        est = cal.step_estimate(prof)
        line["dp_projection"] = {"world": args.profile_world, "busbw_gbs": args.busbw_gbs,
                                 "busbw_source": "nominal (one GPU here)",
                                 "profile": args.profile_out,
                                 "transition_layer": cal.transition_layer(prof),
                                 **{k: v for k, v in est.items()}}
    if args.overlap_bwd > 0:
        line["overlap"] = overlap_bwd(args, items, layers, L, lsp, torch, dev, comm, gdt)
    fit_every = args.fit_every if args.fit_every is not None else (
        100 if args.config == "c3" else 0)
    if fit_every > 0 and rank == 0:
        args.fit_every = fit_every
        line["fit"] = fit_leg(args, items, L, shapes, d, r, lsp, torch, dev)
        line["fit"]["ms_per_step_incl_fit"] = ms + line["fit"]["amortized_ms_per_step"]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb, _ = cpu_baseline(desc, L, shapes, d, r, gdt, args.lr, reps=5)
        line["cpu_baseline"] = cb
    if not args.no_e2e:
        line["e2e"] = e2e(args, items, layers, order, world, dist, torch, dev, bg, comm)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        torch.cuda.synchronize()
        comm.close()  # before the process group and the CUDA context go away
    if world > 1:
        dist.destroy_process_group()


def overlap_bwd(args, items, layers, L, lsp, torch, dev, comm, gdt):
    """North-star subsystem 5 measured: stand-in weight-gradient GEMMs
    (G = X^T dY with args.overlap_bwd token rows; TF32 for fp32 G, bf16 for bf16
    G) produce every layer's gradients on the compute stream, last layer first;
    the LSP chain (compress -> [all-reduce] -> Adam -> Y -> apply) runs on a side
    stream, compress(l) gated by bwd(l)'s event (schedule.py).  Times, per step,
    CUDA-graph replays of (a) the backward alone, (b) backward then the serial
    LSP step, (c) the pipelined step; exposed LSP = (c) - (a)."""
    from paper_2406_10181_b200.schedule import LayerSchedule

    T = args.overlap_bwd
    torch.backends.cuda.matmul.allow_tf32 = True
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[gdt]
    per_layer = len(items) // L
    acts = {}
    gen = torch.Generator(device=dev)
    gen.manual_seed(17)
    for it in items:
        for dim in (it["m"], it["n"]):
            if dim not in acts:
                acts[dim] = torch.randn(T, dim, device=dev, generator=gen).to(tdt)

    def backward(li):
        for it in items[li * per_layer:(li + 1) * per_layer]:
            torch.matmul(acts[it["m"]].t(), acts[it["n"]], out=it["g"])

    order = list(reversed(range(L)))
    serial = LayerSchedule(layers, args.lr, comm=comm)
    lsp_stream = None
    if args.lsp_priority:
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") \
            else (0, -1)
        lsp_stream = torch.cuda.Stream(device=dev, priority=-1)
    piped = LayerSchedule(layers, args.lr, comm=comm, backward=backward, lsp_stream=lsp_stream)
    carve = args.bwd_carveout
    if carve:
        torch._C._set_sm_carveout_experimental(carve)
        lsp.set_sm_budget(carve, carve)

    def bwd_all():
        for li in order:
            backward(li)

    def bwd_then_lsp():
        bwd_all()
        serial.step()

    variants = {"bwd_only": bwd_all, "bwd_then_lsp": bwd_then_lsp, "pipelined": piped.step}
    graphs = {}
    for name, fn in variants.items():
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        graphs[name] = g
    res = {}
    stream = torch.cuda.current_stream()
    for name, g in graphs.items():
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            g.replay()
        t1.record(stream)
        torch.cuda.synchronize()
        res[name] = t0.elapsed_time(t1) / args.steps
    if carve:
        torch._C._set_sm_carveout_experimental(None)
        lsp.set_sm_budget(args.sms_compress, args.sms_update)
    lsp_serial = res["bwd_then_lsp"] - res["bwd_only"]
    exposed = res["pipelined"] - res["bwd_only"]
    out = {"tokens": T, "gemm": "tf32" if gdt == "f32" else "bf16", "carveout_sms": carve,
           "lsp_stream_priority": "high" if args.lsp_priority else "default",
           "bwd_only_ms": res["bwd_only"], "bwd_then_lsp_ms": res["bwd_then_lsp"],
           "pipelined_ms": res["pipelined"], "lsp_serial_ms": lsp_serial,
           "exposed_lsp_ms": exposed,
           "hidden_frac": (1.0 - exposed / lsp_serial) if lsp_serial > 0 else None,
           "note": "CUDA-graph replays; exposed = pipelined - backward alone"}
    if args.timeline_out:
        out["timeline"] = args.timeline_out
        write_timeline(args.timeline_out, piped, torch, T)
    return out


def write_timeline(path, sched, torch, T):
    """One eager pipelined step with CUDA events around every stage on the stream
    it runs on: per-stream start/end times (ms from the step start) as JSON."""
    evs = []
    start = torch.cuda.Event(enable_timing=True)

    def rec(ph, li, when):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())
        evs.append((ph, li, when, e, torch.cuda.current_stream().stream_id))

    sched.record = rec
    torch.cuda.synchronize()
    start.record(torch.cuda.current_stream())
    sched.step()
    torch.cuda.synchronize()
    sched.record = None
    spans = {}
    for ph, li, when, e, sid in evs:
        spans.setdefault((ph, li, sid), {})[when] = start.elapsed_time(e)
    rows = [{"phase": ph, "layer": li, "stream": sid, "begin_ms": v.get("begin"),
             "end_ms": v.get("end")} for (ph, li, sid), v in spans.items()]
    rows.sort(key=lambda x: x["begin_ms"])
    with open(path, "w") as f:
        json.dump({"tokens": T, "spans": rows}, f, indent=1)


def fit_leg(args, items, L, shapes, d, r, lsp, torch, dev):
    """BASELINE configs[2]'s "projector fit every 100 steps": one maybe_update
    (trainer.cpp:74-112: relative-bias gate at alpha 0.5, fresh pair, fit on
    the gradient plus args.fit_ring ring gradients with the reference FitConfig
    defaults -- <= 500 GD steps with line search --, reproject the moments) per
    distinct matrix shape, timed on the device; amortised over the cadence."""
    every = args.fit_every
    per = []
    gen = torch.Generator(device=dev)
    gen.manual_seed(23)
    seen = set()
    for it in items:
        key = (it["m"], it["n"])
        if key in seen:
            continue
        seen.add(key)
        cnt = sum(c for (m, n, c) in shapes if (m, n) == key) * L
        ring = [torch.randn(it["m"], it["n"], device=dev, generator=gen).to(it["g"].dtype)
                for _ in range(args.fit_ring)]
        adam = lsp.AdamState(d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        newp, res = lsp.maybe_update(it["pair"], adam, it["g"], ring, r=r, alpha=0.5,
                                     fit=lsp.FitConfig(), reinit_seed=len(per) + 1)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        per.append({"shape": list(key), "matrices": cnt, "maybe_update_ms": ms,
                    "refreshed": bool(res["refreshed"]), "fit_steps": int(res["fit_steps"]),
                    "fit_timed_out": bool(res["fit_timed_out"]),
                    "bias_before": res["bias_before"], "bias_after": res["bias_after"]})
        del ring
    per_check = sum(x["maybe_update_ms"] * x["matrices"] for x in per)
    return {"every": every, "targets": 1 + args.fit_ring, "per_shape": per,
            "ms_per_check": per_check, "amortized_ms_per_step": per_check / every,
            "note": ("fp64 device fit (csrc/fit.cu); one maybe_update per shape timed, "
                     "times the shape's matrix count; not part of the grad GB/s metric")}


def e2e(args, items, layers, order, world, dist, torch, dev, bg, comm=None):
    """Same metric through the C-ABI with HOST gradients: every step copies each
    layer's G matrices from pinned host memory (copy stream, double-buffered per
    layer) into the bound device buffers, runs the layer step, and reads the
    layer's (all-reduced) S back to pinned host memory."""
    per_layer = len(items) // len(layers)
    host = {}
    for it in items:
        key = (it["m"], it["n"])
        if key not in host:
            h = torch.empty(it["m"], it["n"], dtype=it["g"].dtype, pin_memory=True)
            h.copy_(torch.randn(it["m"], it["n"]).to(it["g"].dtype))
            host[key] = h
    s_host = [torch.empty(tuple(l.s_buffer().shape), dtype=l.s_buffer().dtype, pin_memory=True)
              for l in layers]
    main = torch.cuda.current_stream()
    copy = torch.cuda.Stream(device=dev)
    steps = max(1, min(args.steps, 3))

    def h2d(li):
        with torch.cuda.stream(copy):
            copy.wait_stream(main)  # the layer's G buffers are free (previous compress done)
            for it in items[li * per_layer:(li + 1) * per_layer]:
                it["g"].copy_(host[(it["m"], it["n"])], non_blocking=True)
            e = torch.cuda.Event()
            e.record(copy)
        return e

    def run_step():
        nxt = h2d(order[0])
        for j, li in enumerate(order):
            e = nxt
            if j + 1 < len(order):
                nxt = h2d(order[j + 1])
            main.wait_event(e)
            lay = layers[li]
            if comm is not None:
                lay.compress()
                lay.allreduce(comm)
                lay.update(args.lr)
            else:  # single rank: Adam in the stage-2 epilogue, as in the timed step
                lay.compress_adam()
                lay.apply(args.lr)
            s_host[li].copy_(lay.s_buffer(), non_blocking=True)
        torch.cuda.synchronize()

    run_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        run_step()
    if world > 1:
        dist.barrier()
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        tt = torch.tensor([dt], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    gbytes = sum(it["m"] * it["n"] for it in items) * bg
    return {"value": world * gbytes / dt / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": int(gbytes),
            "d2h_bytes_per_step": int(sum(l.s_buffer().numel() * l.s_buffer().element_size()
                                          for l in layers)),
            "ms_per_step": dt * 1e3, "steps": steps,
            "note": "wall clock incl. H2D of every G from pinned host memory and D2H of every S"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
