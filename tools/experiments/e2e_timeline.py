"""Per-column %globaltimer timeline of the c1 pipelined host path (variants
as in e2e_ablate.py) against the resident path: where the extra time lands."""
import inspect, json, sys, textwrap
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
import paper_2011_05090_b200.gram_schmidt as gsm  # noqa: E402
from paper_2011_05090_b200 import _lib  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device  # noqa: E402

cfg = CONFIGS["c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
pol = sg.policy_from_name(cfg["policy"])
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
Wt = make_w_device(n, m, cfg["sigma_min"], 0, torch.float32, "cuda")
th.device_data(torch.device("cuda", 0))
pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
pin.copy_(Wt[:, :n])
gsm._ABL_WD = Wt[:, :n].contiguous()
Wh = pin.numpy().T
src = textwrap.dedent(inspect.getsource(gsm.RgsState.factorize_host_pipelined))


def variant(no_h2d=False, no_d2h=False):
    s = src
    if no_h2d:
        s = s.replace("Wd = torch.empty((m, n), dtype=dt, device=self.device)", "Wd = _ABL_WD")
        s = s.replace("Wd[c0:c1].copy_(Wt[c0:c1], non_blocking=True)", "pass")
    if no_d2h:
        s = s.replace("Qh[c0:c1].copy_(self._Q[c0:c1, :n], non_blocking=True)", "pass")
    ns = {}
    exec(compile(s, "<variant>", "exec"), gsm.__dict__, ns)
    return ns["factorize_host_pipelined"]


def stamps(run):
    run()
    torch.cuda.synchronize()
    tl = torch.zeros((m + 1, 16), dtype=torch.int64, device="cuda")
    tl[:, 0] = 2**62
    tl[:, 1] = 2**62
    _lib.load().sgs_debug_timeline(tl.data_ptr())
    run()
    torch.cuda.synchronize()
    _lib.load().sgs_debug_timeline(None)
    t = tl.cpu().numpy().astype(np.float64) / 1e3
    go = t[1:m, 1] - t[1, 1]   # column kernel i past its wait, from column 1
    return go, t


def resident():
    st = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=0.0)
    st.factorize_columns(gsm._ABL_WD.T if False else Wt, Wt.shape[1], m)


out = {}
go_res, _ = stamps(resident)
out["resident"] = go_res
for name, kw in [("neither", {"no_h2d": True, "no_d2h": True}), ("full", {})]:
    gsm.RgsState.factorize_host_pipelined = variant(**kw)
    go, t = stamps(lambda: sg.rgs_factorize(Wh, th, pol, with_certificate=False, breakdown_factor=0.0))
    out[name] = go
res = {}
marks = [1, 2, 4, 8, 16, 32, 64, 100, 150, 192, 200, 256, 300, 400, 498]
for name, go in out.items():
    res[name] = {f"c{c}": round(float(go[c - 1]), 1) for c in marks}
# per-column period differences (neither - resident), and where they concentrate
d = np.diff(out["neither"]) - np.diff(out["resident"])
res["neither_minus_resident_period_top"] = sorted(
    [(int(i + 2), round(float(v), 1)) for i, v in enumerate(d)], key=lambda x: -x[1])[:40]
res["neither_minus_resident_period_mean_by_100"] = [round(float(x.mean()), 2) for x in np.array_split(d, 5)]
d = np.diff(out["full"]) - np.diff(out["resident"])
res["full_minus_resident_period_top"] = sorted(
    [(int(i + 2), round(float(v), 1)) for i, v in enumerate(d)], key=lambda x: -x[1])[:60]
res["full_minus_resident_period_sum_by_50"] = [round(float(x.sum()), 1) for x in np.array_split(d, 10)]
print(json.dumps(res))
