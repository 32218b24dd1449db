"""BASELINE configs[4]: the d x r sweep on 4096 x 11008 (fp32), one bench.py run
per point (CUDA-graph replay, --c5-layers independent matrices per step so the
inputs exceed L2), collected into one JSON document with the per-point
roofline of the dominant kernel (k_apply_y) and the compress phase.

    python tools/c5_grid.py OUT.json [--d 256,512,...] [--r 2,4,8]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--d", default="256,512,1024,2048,4096")
    ap.add_argument("--r", default="2,4,8")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    points = []
    for d in [int(x) for x in a.d.split(",")]:
        for r in [int(x) for x in a.r.split(",")]:
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c5", "--d", str(d),
                   "--r", str(r), "--steps", str(a.steps), "--warmup", "3", "--no-e2e",
                   "--no-cpu-baseline"]
            p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
            if p.returncode != 0:
                points.append({"d": d, "r": r, "error": p.stderr.strip().splitlines()[-1:]})
                print(d, r, "FAILED", p.stderr.strip().splitlines()[-1:], flush=True)
                continue
            x = json.loads(p.stdout.strip().splitlines()[-1])
            b = x["breakdown"]
            pt = {"d": d, "r": r, "ms_per_step": x["ms_per_step"], "grad_gbs": x["value"],
                  "matrices": x["config"]["matrices"],
                  "step_hbm_frac_of_measured": x["config"]["step_hbm_frac_of_measured"],
                  "apply_frac": x["roofline"]["frac"], "apply_gbs": x["roofline"]["achieved"],
                  "compress_frac": b["compress_frac"], "compress_gbs": b["compress_achieved_gbs"],
                  "phase_ms_per_step": {k[:-12]: v for k, v in b.items() if k.endswith("ms_per_step")},
                  "clocks": x.get("clocks")}
            points.append(pt)
            print(json.dumps(pt), flush=True)
    doc = {"config": "BASELINE configs[4]: 4096 x 11008 fp32, d x r grid (d = subspace width, "
                     "r = nonzeros per projector row; BASELINE.json swaps the letters)",
           "peak_gbs": points[0].get("apply_gbs") and None, "points": points}
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
