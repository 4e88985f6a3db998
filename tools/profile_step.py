"""Per-kernel timeline of one RGS-QR factorisation (CUPTI via torch.profiler):
kernel time per class, and idle gaps on the stream between kernels.

    python tools/profile_step.py [--config c1] [--m M]
"""

import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2011_05090_b200 as sg
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--out", default="gpurun_out/profile_step.json")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    n, m, k = cfg["n"], args.m or cfg["m"], cfg["k"]
    pol = sg.policy_from_name(cfg["policy"])
    kw = {"block_log2": cfg["block_log2"]} if "block_log2" in cfg else {}
    th = sg.make_sketch(sg.SketchKind(cfg["kind"]), k, n, 0, **kw)
    wdt = torch.float32 if pol.coarse_dtype == np.float32 else torch.float64
    Wt = make_w_device(n, m, cfg["sigma_min"], 0, wdt, "cuda")
    th.device_data()

    def step():
        st = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=cfg["breakdown_factor"])
        st.factorize_columns(Wt, Wt.shape[1], m)

    step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs
                   if "Memcpy" not in e.name and "Memset" not in e.name])
    agg = collections.defaultdict(lambda: [0, 0.0])
    gaps = []
    for j, (s, e, name) in enumerate(kern):
        key = name.split("<")[0].replace("void ", "").replace("sgs::", "")
        agg[key][0] += 1
        agg[key][1] += e - s
        if j:
            gaps.append(max(0.0, s - kern[j - 1][1]))
    span = kern[-1][1] - kern[0][0]
    out = {"config": args.config, "m": m, "span_us": span,
           "kernels": {k2: {"n": v[0], "total_us": round(v[1], 1), "avg_us": round(v[1] / v[0], 2),
                            "share": round(v[1] / span, 4)} for k2, v in agg.items()},
           "gaps_total_us": round(sum(gaps), 1),
           "gap_avg_us": round(sum(gaps) / max(1, len(gaps)), 2),
           "gap_p50_us": round(float(np.median(gaps)), 2) if gaps else 0}
    # per-column trend of the LS kernel
    ls = [(e - s) for s, e, nm in kern if "ls_step" in nm]
    if ls:
        out["ls_us_by_decile"] = [round(float(np.mean(c)), 2) for c in np.array_split(ls, 10)]
    sr = [(e - s) for s, e, nm in kern if "srht" in nm or "dense" in nm]
    if sr:
        out["sketch_us_by_decile"] = [round(float(np.mean(c)), 2) for c in np.array_split(sr, 10)]
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
