"""c1 pipelined host path: per chunk, when W landed (H2D event), when its sketch
finished (side stream) and when the compute stream passed its wait - is the
compute stream waiting on PCIe or the other way round?"""
import inspect, json, sys, textwrap
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2011_05090_b200 as sg  # noqa: E402
import paper_2011_05090_b200.gram_schmidt as gsm  # noqa: E402
from paper_2011_05090_b200.workloads import CONFIGS, make_w_device  # noqa: E402

cfg = CONFIGS["c1"]
n, m, k = cfg["n"], cfg["m"], cfg["k"]
pol = sg.policy_from_name(cfg["policy"])
th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
Wt = make_w_device(n, m, cfg["sigma_min"], 0, torch.float32, "cuda")
th.device_data(torch.device("cuda", 0))
pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
pin.copy_(Wt[:, :n])
del Wt
torch.cuda.empty_cache()
Wh = pin.numpy().T
s = textwrap.dedent(inspect.getsource(gsm.RgsState.factorize_host_pipelined))
s = s.replace("torch.cuda.Event()", "torch.cuda.Event(enable_timing=True)")
s = s.replace("landed.append(ev)", "landed.append(ev); _ABL['landed'].append(ev); _ABL['copy_host'].append(__import__('time').perf_counter())")
s = s.replace("sketched.append(ev)", "sketched.append(ev); _ABL['sketched'].append(ev)")
s = s.replace("comp.wait_event(sketched[int(chunk_of[nxt])])",
              "comp.wait_event(sketched[int(chunk_of[nxt])]); _e = torch.cuda.Event(enable_timing=True); "
              "_e.record(comp); _ABL['passed'].append((i, _e))")
s = s.replace("self.status.reset()", "_mark('pre_reset'); self.status.reset(); _mark('reset')")
s = s.replace("comp.wait_event(sketched[0])", "_mark('pre_w0'); comp.wait_event(sketched[0]); _mark('w0')")
s = s.replace("Wd = torch.empty((m, n), dtype=dt, device=self.device)",
              "_mark('fn_entry'); Wd = torch.empty((m, n), dtype=dt, device=self.device)")


def _mark(tag):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    gsm._ABL["early"].append((tag, e))


gsm._mark = _mark
s = s.replace("Qh[c0:c1].copy_(self._Q[c0:c1, :n], non_blocking=True)",
              "_s0 = torch.cuda.Event(enable_timing=True); _s0.record(); "
              "Qh[c0:c1].copy_(self._Q[c0:c1, :n], non_blocking=True); "
              "_s1 = torch.cuda.Event(enable_timing=True); _s1.record(); _ABL['ship'].append((c0, c1, _s0, _s1))")
assert "_ABL['passed']" in s
ns = {}
exec(compile(s, "<variant>", "exec"), gsm.__dict__, ns)
gsm.RgsState.factorize_host_pipelined = ns["factorize_host_pipelined"]
out = {}
_oc, _ol = gsm.RgsState._column, gsm.RgsState._ls


def _col(self, i, *a, **kw):
    r = _oc(self, i, *a, **kw)
    if i < 6:
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        gsm._ABL["early"].append((f"col{i}", e))
    return r


def _ls(self, **kw):
    r = _ol(self, **kw)
    if kw.get("fin") is not None and kw["fin"] < 6:
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        gsm._ABL["early"].append((f"ls{kw['fin']}", e))
    return r


gsm.RgsState._column, gsm.RgsState._ls = _col, _ls
f = None
res = {}
for rep in range(6):
    gsm.RgsState._e2e_ahead = 4 if rep % 2 == 0 else 100
    f = None  # pinned result buffers are reused only once released
    gsm._ABL = {"landed": [], "sketched": [], "passed": [], "early": [], "copy_host": [], "ship": []}
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = __import__("time").perf_counter()
    f, _ = sg.rgs_factorize(Wh, th, pol, with_certificate=False, breakdown_factor=0.0)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    torch.cuda.synchronize()
    A = gsm._ABL
    out = {"total_ms": e0.elapsed_time(e1), "host_ms": 1e3 * (__import__("time").perf_counter() - h0),
           "landed_ms": [round(e0.elapsed_time(e), 3) for e in A["landed"]],
           "sketched_ms": [round(e0.elapsed_time(e), 3) for e in A["sketched"]],
           "passed": [(i, round(e0.elapsed_time(e), 3)) for i, e in A["passed"]],
           "copy_host_ms": [round(1e3 * (t - h0), 3) for t in A["copy_host"]],
           "ship": [(a, b, round(e0.elapsed_time(x), 3), round(e0.elapsed_time(y), 3)) for a, b, x, y in A["ship"]],
           "early": [(t, round(e0.elapsed_time(e), 3)) for t, e in A["early"]]}
    res[f"rep{rep}_ahead{gsm.RgsState._e2e_ahead}"] = out
print(json.dumps(res))
