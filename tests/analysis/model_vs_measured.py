"""Predicted vs measured, from the committed sweeps.

For every measured point in profiles/r01_sweep_n*.jsonl:
- The reference's own closed-form prediction: oracle/_ref simulate_exchange on
  the nvswitch model at 900 GB/s per port, default PipelineConfig.
- The measured time.
- A B200 calibration: measured time is modelled as t0 + port_bytes / B_eff,
  fitted by least squares over all points >= 64 MiB.  B_eff is the effective
  per-port rate the planner's link-load model should use on this box.

Writes profiles/r01_model_vs_measured.md.  Needs oracle/_ref (build container).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2604_00317_b200 import planner as P  # noqa: E402

MiB = 1 << 20


def matrix_for(row):
    R = row["ranks"]
    if row["case"] == "c3":
        return P.gen_skewed_a2av(R, 256 * MiB, row["ratio"], 0)
    if row["case"] == "c5":
        return P.gen_skewed_a2av(R, 256 * MiB, 1.0 / (R - 1), 0)
    if row["case"] == "c4":
        return P.gen_irregular(R, row["total"], 0.5, 1)
    if row["case"] == "c1":
        return P.gen_p2p(R, 0, 1, 64 * MiB)
    return P.gen_p2p(R, 0, 1, 1 << 30)


def port_bytes(m, R):
    return max(max(sum(m[v * R + d] for d in range(R) if d != v), sum(m[s * R + v] for s in range(R) if s != v))
               for v in range(R))


def main():
    rows = []
    for n in (2, 3, 4):
        path = os.path.join(ROOT, "profiles", f"r01_sweep_n{n}.jsonl")
        if os.path.exists(path):
            rows += [json.loads(x) for x in open(path) if x.startswith("{")]
    out = ["# Reference model vs B200 measurement (round 1)", "",
           "- `model_us`: the reference's `simulate_exchange` closed-form prediction. It runs on the",
           "  nvswitch model at 900 GB/s per port with the default PipelineConfig, through oracle/_ref.",
           "- `measured_us`: the median from `tools/sweeps.py` on 2-4 B200s.", "",
           "| case | W | model | measured_us | model_us | measured/model | port MB |", "|---|---|---|---|---|---|---|"]
    fit = []
    for r in rows:
        R = r["ranks"]
        m = matrix_for(r)
        fab = r.get("fabric_model", "nvswitch")
        req = {"ranks": R, "topology": {"nodes": 1, "gpus": R, "nics": 0, "fabric": fab, "nvlink_gbps": 900.0,
                                        "rail_gbps": 50.0}, "workload": {"kind": "matrix", "bytes": m}}
        model = ref.call(dict(req, op="simulate"))["completion"] * 1e6
        pb = port_bytes(m, R)
        tag = r["case"] + (f" r={r['ratio']}" if "ratio" in r else "") + (f" T={r['total']}" if "total" in r else "")
        out.append(f"| {tag} | {R} | {fab} | {r['us']:.1f} | {model:.1f} | {r['us'] / model:.2f} | {pb / 1e6:.1f} |")
        if pb >= 64 * MiB and fab == "nvswitch":
            # one-way: the busiest port's reverse direction carries < half as much
            rev = max(min(sum(m[v * R + d] for d in range(R) if d != v), sum(m[s * R + v] for s in range(R) if s != v))
                      for v in range(R) if max(sum(m[v * R + d] for d in range(R) if d != v),
                                               sum(m[s * R + v] for s in range(R) if s != v)) == pb)
            fit.append((pb, r["us"] * 1e-6, "one-way" if rev < pb / 2 else "two-way"))
    out += ["", "## B200 calibration", "",
            "Least squares t = t0 + port_bytes / B_eff over nvswitch points with >= 64 MiB on the busiest port.",
            "Points are split by whether that port's reverse direction carries less than half as much",
            "(one-way: p2p, skewed hot port) or not (two-way: uniform, mild skew).", "",
            "| class | points | B_eff GB/s | t0 us | max rel. residual |", "|---|---|---|---|---|"]
    best = None
    for cls in ("one-way", "two-way"):
        pts = [(x, y) for x, y, c in fit if c == cls]
        n = len(pts)
        if n < 2:
            continue
        sx, sy = sum(x for x, _ in pts), sum(y for _, y in pts)
        sxx, sxy = sum(x * x for x, _ in pts), sum(x * y for x, y in pts)
        slope = (n * sxy - sx * sy) / (n * sxx - sx * sx)
        t0 = (sy - slope * sx) / n
        resid = max(abs(t0 + slope * x - y) / y for x, y in pts)
        out.append(f"| {cls} | {n} | {1 / slope / 1e9:.0f} | {t0 * 1e6:.1f} | {resid:.3f} |")
        if cls == "one-way":
            best = 1 / slope
    out += ["",
            "The reference's model assumes 900 GB/s of user data per port and 2 us per hop. On B200 the fitted "
            "rates sit below that by the NVLink protocol overhead (16 B per 128 B for pulls, 24 B for pushes; "
            "`profiles/r01_summary.md`) plus per-call fixed cost. "
            f"Feeding B_eff = {best / 1e9:.0f} GB/s into the planner (`nimbleCommConfig.nvlink_bytes_per_s`) makes its "
            "link-load model B200-truthful for one-way ports. Routing does not change on the nvswitch model: "
            "the plan is direct either way."]
    with open(os.path.join(ROOT, "profiles", "r01_model_vs_measured.md"), "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out[-8:]))


if __name__ == "__main__":
    main()
