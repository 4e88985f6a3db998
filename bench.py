"""Benchmark: RGS-QR columns/s on BASELINE config 1 (and other configs on request).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1]
    python bench.py --impl reference ...        # CPU reference arm (oracle port)
    torchrun --nproc-per-node N bench.py --gpus N   # row-sharded, NCCL all-reduce

A step is one full randomized Gram-Schmidt factorisation of the config's W
(n x m) already resident in HBM (``value``), or through the public API from
pinned host memory with the factors copied back (``e2e``).  Rank 0 prints one
JSON line.  W and Q (2 GB each at c1) exceed the 126 MB L2, so no flush is
needed between steps.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, gpu: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def _traffic(cfg_name):
    """(DRAM bytes of one launch of the dominant kernel from the committed ncu
    --set full capture, note) for a config, or (None, None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as fh:
            tj = json.load(fh).get(cfg_name)
    except (OSError, ValueError):
        tj = None
    if not tj:
        return None, None
    return tj["dram_bytes"], (f"ncu --set full, {tj['kernel']} at column {tj['column']}: "
                              f"{tj['dram_bytes']:.4g} B DRAM vs {tj['alg_bytes']:.4g} B "
                              f"algorithmic ({tj['source']})")


def qr_alg_bytes(n, m, bq, bw, k=0, gaussian=False):
    """n b_Q m(m+1)/2 + 2 n b_W m (+ (m+1) k n 8 for Gaussian)."""
    b = n * bq * m * (m + 1) / 2 + 2 * n * bw * m
    if gaussian:
        b += (m + 1) * k * n * 8
    return b


def update_alg_bytes(n, i, bq, bw):
    """One sgs_rgs_update launch for column i: read Q[:, :i], read w, write q'_i,
    write the normalised q_{i-1} (i > 0)."""
    return n * bq * i + n * bw + n * bq + (n * bq if i > 0 else 0)


# ---------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _oracle_problem(cfg, n_cols, threads):
    from oracle import OracleSketch
    from paper_2011_05090_b200.workloads import make_w
    n, k = cfg["n"], cfg["k"]
    W = make_w(n, n_cols, cfg["sigma_min"], 0,
               dtype=np.float32 if cfg["policy"] == "mixed" else np.float64, threads=threads)
    th = OracleSketch(cfg["kind"], k, n, 0, threads=threads,
                      **({"block_log2": cfg["block_log2"]} if "block_log2" in cfg else {}))
    return W, th


def cpu_sample(cfg, n_cols, threads):
    """Time the oracle port (the reference's algorithm, reference numerics) on
    the first n_cols columns of a config-shaped problem."""
    from threadpoolctl import threadpool_limits
    from oracle import OracleRgs
    W, th = _oracle_problem(cfg, n_cols, threads)
    with threadpool_limits(limits=threads, user_api="blas"):
        st = OracleRgs(th, cfg["policy"], cfg["breakdown_factor"], capacity=n_cols)
        t0 = time.perf_counter()
        for j in range(n_cols):
            st.push(W[:, j])
        dt = time.perf_counter() - t0
    return n_cols / dt, dt


def cpu_baseline_block(cfg_name, cfg, all_cols, one_cols):
    """cpu_baseline of the GPU arm: the oracle port on the first columns of the
    config's problem with every host thread, and (BASELINE.md section 3,
    SURVEY 8(d)) with one BLAS thread ("1 core")."""
    threads = os.cpu_count() or 1
    v, dt = cpu_sample(cfg, all_cols, threads)
    v1, dt1 = cpu_sample(cfg, one_cols, 1)
    return {"value": v, "unit": "columns/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"first {all_cols} columns of {cfg_name} (n={cfg['n']}, k={cfg['k']} "
                      f"{cfg['kind']}, {cfg['policy']}), oracle port of sketchgs, "
                      f"{threads} threads, {dt:.1f} s (early columns: the full run is the "
                      f"reference arm, bench.py --impl reference)",
            "one_core": {"value": v1, "unit": "columns/s", "cores": 1,
                         "sample": f"first {one_cols} columns, OPENBLAS 1 thread, {dt1:.1f} s"}}


def qr_config(cfg_name, cfg, n, m, k, world, suffix=""):
    """The `config` object of an RGS-QR bench line (both arms emit exactly this)."""
    return {"workload": cfg_name + suffix, "n": n, "m": m, "k": k, "sketch": cfg["kind"],
            "policy": cfg["policy"], "breakdown_factor": cfg["breakdown_factor"],
            "parallelism": f"row-shard x{world}" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (W, Q >> 126 MB)"}


# full factorisations the reference arm can time within a few minutes on the
# GPU box's host (c1: ~2.5 min on 16 threads); larger configs time a prefix
REF_FULL = {"c0", "c0r", "c1"}


def run_reference(args, cfg_name):
    """The reference arm: the oracle port of sketchgs (pinned bit for bit to the
    reference by tests/test_oracle_golden.py) on the host cores, same config,
    metric and unit as our arm.  For c0/c1 the K timed steps are K consecutive
    segments of ONE full factorisation of the config's W (value = m / total
    time: late columns cost more, so a prefix would flatter the CPU); warm-up
    steps push columns into a throwaway state.  Generation of W and Theta is
    excluded."""
    import torch  # noqa: F401  (keeps the import cost out of the timed region)
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if cfg_name == "c3":
        return run_reference_gmres(args)
    from threadpoolctl import threadpool_limits
    from oracle import OracleRgs
    from paper_2011_05090_b200.workloads import CONFIGS
    cfg = CONFIGS[cfg_name]
    threads = os.cpu_count() or 1
    world = max(1, args.gpus)
    m = args.columns if args.columns is not None else cfg["m"]
    full = cfg_name in REF_FULL or args.columns is not None
    m_run = m if full else min(m, args.cpu_cols)
    t_gen = time.perf_counter()
    W, th = _oracle_problem(cfg, m_run if full else m_run, threads)
    t_gen = time.perf_counter() - t_gen
    K = max(1, min(args.steps, m_run))
    bounds = [(m_run * s) // K for s in range(K + 1)]
    times = []
    with threadpool_limits(limits=threads, user_api="blas"):
        warm = OracleRgs(th, cfg["policy"], cfg["breakdown_factor"], capacity=max(1, args.warmup))
        for j in range(min(args.warmup, m_run)):
            warm.push(W[:, j])
        del warm
        st = OracleRgs(th, cfg["policy"], cfg["breakdown_factor"], capacity=m_run)
        for s in range(K):
            t0 = time.perf_counter()
            for j in range(bounds[s], bounds[s + 1]):
                st.push(W[:, j])
            times.append(time.perf_counter() - t0)
    total = sum(times)
    v = m_run / total
    what = (f"one full {cfg_name} factorisation ({m_run} columns) in {K} consecutive segments"
            if full else f"first {m_run} of {m} columns of {cfg_name} in {K} segments "
                         f"(the full run exceeds the bench budget)")
    sample = (f"{what}, oracle port of sketchgs (numpy/OpenBLAS, {threads} threads), "
              f"{total:.1f} s timed, W/Theta generation {t_gen:.1f} s excluded")
    print(json.dumps({
        "impl": "reference", "metric": "RGS-QR columns/s", "value": v, "unit": "columns/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (Q, update) / f64 (sketch, LS)" if cfg["policy"] == "mixed" else "f64",
        "data": "synthetic (W = G diag(sigma) V^T, seeded numpy Philox)",
        "config": qr_config(cfg_name, cfg, cfg["n"], m, cfg["k"], world,
                            "" if args.columns is None else f"-m{m}"),
        "columns_timed": m_run, "segment_s": [round(t, 3) for t in times],
        "cpu_baseline": {"value": v, "unit": "columns/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": v, "unit": "columns/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def run_reference_gmres(args):
    """Reference arm of c3: the oracle port's RGS-Arnoldi steps on the full
    128^3 operator (SpMV, two P-SRHT applies and the Householder LS per step,
    reference numerics).  A whole 549-iteration solve takes ~10 min on the
    host, so each timed step is a bounded run of consecutive Arnoldi steps of
    the first cycle."""
    from threadpoolctl import threadpool_limits
    from oracle import OracleRgs, OracleSketch, csr_matvec
    from paper_2011_05090_b200.workloads import CONFIGS, convdiff3d, rhs_gaussian
    cfg = CONFIGS["c3"]
    threads = os.cpu_count() or 1
    N = cfg["grid"]
    rp, ci, va = convdiff3d(N, (cfg["beta"],) * 3)
    n = N ** 3
    b = rhs_gaussian(n, 0)
    th = OracleSketch("psrht", cfg["k"], n, 0)
    K = max(1, args.steps)
    per = max(1, 60 // K)
    times = []
    with threadpool_limits(limits=threads, user_api="blas"):
        st = OracleRgs(th, "f64", capacity=K * per + args.warmup + 2)
        st.push(b / np.linalg.norm(b))
        i = 0
        for _ in range(args.warmup):
            st.push(csr_matvec(rp, ci, va, n, st.Q[:, i].astype(np.float64)))
            i += 1
        for _ in range(K):
            t0 = time.perf_counter()
            for _ in range(per):
                st.push(csr_matvec(rp, ci, va, n, st.Q[:, i].astype(np.float64)))
                i += 1
            times.append(time.perf_counter() - t0)
    total = sum(times)
    v = K * per / total
    print(json.dumps({
        "impl": "reference", "metric": "RGMRES Arnoldi steps/s", "value": v, "unit": "steps/s",
        "n_gpus": max(1, args.gpus), "steps": K, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c3", **cfg, "l2": "inputs larger than L2 (basis, CSR >> 126 MB)"},
        "cpu_baseline": {"value": v, "unit": "steps/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"Arnoldi steps {args.warmup + 1}..{i} of the first cycle "
                                   f"({per} per timed step), fp64 basis, oracle port"},
        "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
def run_qr(args, cfg_name, comm):
    """One config's bench line (a dict on rank 0, None elsewhere)."""
    import torch
    import paper_2011_05090_b200 as sg
    from paper_2011_05090_b200 import _lib
    from paper_2011_05090_b200.workloads import CONFIGS, make_w_device, shard_rows

    rank = comm.rank if comm else 0
    world = comm.world if comm else 1
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = CONFIGS[cfg_name]
    n, m, k = cfg["n"], cfg["m"], cfg["k"]
    if cfg_name == "c4" and world < 4 and args.columns is None:
        # W and Q are 201 GB each in fp32 (BASELINE configs[4]: 4 and 8 GPUs only)
        return {"metric": "RGS-QR columns/s", "impl": "ours", "n_gpus": world,
                "unavailable": "c4 needs >= 4 GPUs (W and Q are 201 GB each)"}
    if args.columns is not None:  # functional runs of a config's shapes with fewer columns
        m = args.columns
    pol = sg.policy_from_name(cfg["policy"])
    bf = cfg["breakdown_factor"]
    kw = {"block_log2": cfg["block_log2"]} if "block_log2" in cfg else {}
    # N > 1: c1 is weak-scaled (n = N x 1e6 rows, ~1e6 per GPU, one P-SRHT over
    # next_pow2(n)); the fixed-n configs (c0, c2) are strong-scaled row shards.
    weak = world > 1 and args.scaling == "weak" and cfg["kind"] == "psrht"
    n_per_gpu = n
    if weak:
        n = n_per_gpu * world
    th = sg.make_sketch(sg.SketchKind(cfg["kind"]), k, n, 0, **kw)
    row0, n_loc = (0, n) if world == 1 else shard_rows(n, world, rank, th.row_align())
    wdt = torch.float32 if pol.coarse_dtype == np.float32 else torch.float64
    Wt = make_w_device(n, m, cfg["sigma_min"], 0, wdt, dev, row0=row0, n_local=n_loc)
    ldw = Wt.shape[1]
    th.device_data(dev)
    torch.cuda.synchronize()

    # one device state for every step (W and Q of c2 are 67 GB each)
    gstate = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=bf, comm=comm, row0=row0,
                         n_local=n_loc)

    def step():
        gstate.m = 0
        gstate.factorize_columns(Wt, ldw, m)
        return gstate

    # the timed steps replay one CUDA graph of the whole factorisation (every
    # kernel re-runs; the graph only removes host launch overhead).  A sharded
    # state captures its NCCL all-reduces too, after one eager factorisation
    # has brought the communicator up (gloo is host-side: no graph).
    graph = None
    graph_launches = 0
    if not args.no_graph and (comm is None or comm.capturable):
        if comm is not None:
            step()
            torch.distributed.barrier()
            gstate.m = 0
        lcg = _lib.launch_count()
        graph = gstate.capture_factorization(Wt, ldw, m)
        graph_launches = _lib.launch_count() - lcg

    graph_used = graph is not None

    def timed_step():
        if graph is not None:
            graph.replay()
        else:
            step()

    def barrier():
        torch.cuda.synchronize()
        if comm:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    # state allocation is part of a step (RgsState buffers), sync at the end is too
    for _ in range(args.warmup):
        timed_step()
    barrier()
    if graph is not None:
        gstate.finish()
    lc0 = _lib.launch_count()
    clocks = Clocks(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        timed_step()
    e1.record()
    barrier()
    clk = clocks.stop()
    launches = _lib.launch_count() - lc0
    shard_sum = (None if comm is None else
                 ("peer-memory exchange in the LS launch"
                  if gstate.__dict__.get("_peer") is not None else "nccl all-reduce"))
    if graph is not None:
        gstate.finish()  # raises if the replayed factorisation recorded a breakdown
        launches = graph_launches * args.steps
    ms = e0.elapsed_time(e1) / args.steps
    if comm:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t)
    # weak: every rank factorises its ~1e6-row share of each column, so the
    # work unit is a c1-sized column shard (world of them per column)
    units = m * world if weak else m
    value = units / (ms / 1e3)
    bq = 4 if pol.coarse_dtype == np.float32 else 8
    bw = bq
    alg = qr_alg_bytes(n, m, bq, bw, k, cfg["kind"] == "gaussian")
    hbm_gbs = alg / (ms / 1e3) / 1e9

    # ---- roofline of the dominant kernel (sgs_rgs_update), CUDA events per launch
    peak, peak_kind = _peaks()
    roof = None
    if True:  # every rank: the step holds collectives; rank 0 reports
        import paper_2011_05090_b200.gram_schmidt as gsm
        evs = []
        orig = gsm.RgsState._column

        def timed_column(self, i, w_ptr, w_code, normalize_prev, sketch, **kw_):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = orig(self, i, w_ptr, w_code, normalize_prev, sketch, **kw_)
            b.record()
            evs.append((i, a, b))
            return out

        gsm.RgsState._column = timed_column
        try:
            step()
        finally:
            gsm.RgsState._column = orig
        torch.cuda.synchronize()
        tot_ms = sum(a.elapsed_time(b) for _, a, b in evs)
        tot_b = sum(update_alg_bytes(n_loc, i, bq, bw) for i, _, _ in evs)
        if cfg["kind"] == "gaussian":
            # the timed unit is the update kernel + the dense sketch GEMV of q'
            # (Theta streamed once per column, q' re-read from L2)
            tot_b += sum(k * n_loc * 8 + n_loc * bq for i, _, _ in evs if i > 0)
        elif cfg["kind"] == "rademacher":
            # update kernel + packed-sign sketch of q' (1 bit per entry, q' re-read)
            tot_b += sum(k * n_loc // 8 + n_loc * bq for i, _, _ in evs if i > 0)
        ach = tot_b / (tot_ms / 1e3) / 1e9
        traffic, traffic_note = None, None
        traffic, traffic_note = _traffic(cfg_name)
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "frac_nominal_8tbs": round(ach / 8000.0, 4),
                "traffic": traffic, "traffic_note": traffic_note,
                "kernel": {"gaussian": "dense_ring_kernel (Q + Theta^T through a TMA bulk-copy ring)",
                           "rademacher": "rgs_update_kernel + rademacher_partials_kernel "
                                         "(device-generated packed signs)"}.get(
                    cfg["kind"], "rgs_column_kernel (update + SRHT epilogue)"),
                "peak_source": peak_kind,
                "share_of_step": round(tot_ms / ms, 4),
                "launches": len(evs), "avg_launch_us": round(1e3 * tot_ms / len(evs), 2),
                # Under programmatic dependent launch the events bracket a launch
                # from its predecessor's end: the column kernel's pre-wait prologue
                # (ring prologue + its paced L2 prefetch, ~100 MB of the next
                # columns) overlaps the predecessor LS launch and is not in the
                # duration, so the per-launch figure can exceed the copy peak;
                # hbm_frac_whole_step is the fraction with nothing excluded.
                "note": ("launch durations exclude the pre-wait L2 prefetch that overlaps the "
                         "predecessor LS launch; hbm_frac_whole_step excludes nothing"
                         if cfg["kind"] == "gaussian" or (
                             cfg["kind"] in ("psrht", "block_srht") and (n_loc + 4095) // 4096 <= 296)
                         else "early columns' Q slices fit in L2, so achieved/peak can exceed 1; "
                              "hbm_frac_whole_step excludes nothing")}

    # ---- e2e through the public API (pinned host W -> factors on the host)
    e2e = None
    e2e_note = None
    # pinned host W and host Q (plus R, S, P) per rank: skip the leg when the
    # host cannot hold them with a margin (c4: 50 GB per rank; c2: 62.5 GB)
    import psutil
    # (torch's pinned allocator rounds each buffer up to a power of two)
    buf = 1 << int(np.ceil(np.log2(n_loc * m * (4 if wdt == torch.float32 else 8))))
    need = 2 * buf * (world if comm else 1)
    if not args.no_e2e and psutil.virtual_memory().available < 1.25 * need:
        e2e_note = (f"skipped: pinned host W + Q need {need / 2**30:.0f} GiB, "
                    f"{psutil.virtual_memory().available / 2**30:.0f} GiB available")
    elif not args.no_e2e:
        del graph, gstate
        torch.cuda.empty_cache()
        pin = torch.empty((m, n_loc), dtype=wdt, pin_memory=True)
        pin.copy_(Wt[:, :n_loc])
        del Wt  # c2: the device W (62.5 GB) would not fit next to the call's own W and Q
        torch.cuda.empty_cache()
        Wh = pin.numpy().T  # (n_loc, m) Fortran-ordered numpy view of pinned memory
        kw_sh = {"comm": comm, "row0": row0} if comm else {}

        def e2e_call():
            return sg.rgs_factorize(Wh, th, pol, with_certificate=False, breakdown_factor=bf,
                                    **kw_sh)

        f = None
        for _ in range(2):  # allocates the pinned output buffers once
            f = None  # the previous result's buffers are reused only once released
            f, _ = e2e_call()
        barrier()
        # The interpreter's cyclic collector is off inside the timed calls (as
        # timeit does): a full collection of this process (torch, numpy, scipy
        # imported) takes tens of ms and showed up as one slow call in three
        # (c1 [86.8, 99.3, 87.1] ms, c0 [33.8, 111.7, 50.7] ms).  Reference
        # counting still frees every buffer; nothing of the measured work moves.
        import gc
        gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        ne = max(1, min(args.steps, 3))
        calls_ms = []
        try:
            for _ in range(ne):
                f = None
                tc = time.perf_counter()
                f, _ = e2e_call()
                calls_ms.append(round(1e3 * (time.perf_counter() - tc), 2))
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / ne
        finally:
            gc.enable()
        if comm:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t)
        fb = np.dtype(pol.fine_dtype).itemsize
        e2e = {"value": units / dt, "unit": "columns/s", "h2d_bytes_per_step": n * m * bq,
               "d2h_bytes_per_step": n * m * bq + world * (m * m * 8 + 2 * k * m * fb),
               "ms_per_step": 1e3 * dt, "calls_ms": calls_ms, "python_gc": "disabled in the timed calls",
               "path": "rgs_factorize(pinned host W shard) -> host Q, R, S, P"}
        del pin, Wh, f

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_block(cfg_name, cfg, args.cpu_cols, max(8, args.cpu_cols // 4))
    if rank == 0:
        return {
            "metric": "RGS-QR columns/s", "value": value, "unit": "columns/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak" if weak else "strong",
            "vs_baseline": None,
            "dtype": "f32 (Q, update) / f64 (sketch, LS)" if cfg["policy"] == "mixed" else "f64",
            "data": "synthetic (W = G diag(sigma) V^T generated on device, seeded)",
            "config": {**qr_config(cfg_name, cfg, n, m, k, world,
                                   ("-weak" if weak else "")
                                   + (f"-m{m}" if args.columns is not None else "")),
                       **({"weak": f"n = {world} x {n_per_gpu} rows (~{n_per_gpu} per GPU); "
                                   f"value counts column shards: {world} per column"}
                          if weak else {})},
            "graph": graph_used,
            # how a row-sharded state sums s' per column: inside the LS launch by
            # NVLink stores into the peers' exchange areas, or an NCCL all-reduce
            "shard_sum": shard_sum,
            "hbm_gbs_whole_step": round(hbm_gbs, 1),
            "hbm_frac_whole_step": round(hbm_gbs / (peak * world), 4),
            # BASELINE.json quotes the nominal ~8 TB/s; the roofline uses the measured peak
            "hbm_frac_whole_step_nominal_8tbs": round(hbm_gbs / (8000.0 * world), 4),
            "alg_bytes_per_step": alg,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            **({"e2e_note": e2e_note} if e2e_note else {}), "gpu_launches": launches,
            "clocks": clk,
        }
    return None


def cpu_gmres_sample(n_steps, threads):
    """The oracle port's Arnoldi steps on c3 at full size (SpMV, two P-SRHT
    applies and the LS per step, reference numerics), first steps of a cycle."""
    from threadpoolctl import threadpool_limits
    from oracle import OracleRgs, OracleSketch, csr_matvec
    from paper_2011_05090_b200.workloads import CONFIGS, convdiff3d, rhs_gaussian
    cfg = CONFIGS["c3"]
    N = cfg["grid"]
    rp, ci, va = convdiff3d(N, (cfg["beta"],) * 3)
    n = N ** 3
    b = rhs_gaussian(n, 0)
    th = OracleSketch("psrht", cfg["k"], n, 0)
    with threadpool_limits(limits=threads):
        st = OracleRgs(th, "f64", capacity=n_steps + 2)
        st.push(b / np.linalg.norm(b))
        t0 = time.perf_counter()
        for i in range(n_steps):
            st.push(csr_matvec(rp, ci, va, n, st.Q[:, i].astype(np.float64)))
        dt = time.perf_counter() - t0
    return n_steps / dt, dt


def run_gmres(args):
    import torch
    import paper_2011_05090_b200 as sg
    import paper_2011_05090_b200.gram_schmidt as gsm
    from paper_2011_05090_b200 import _lib
    from paper_2011_05090_b200.distributed import init_from_env
    from paper_2011_05090_b200.workloads import CONFIGS, convdiff3d, rhs_gaussian
    comm = init_from_env(os.environ.get("SGS_DIST_BACKEND", "nccl"))
    if comm is not None:
        return run_gmres_sharded(args, comm)
    cfg = CONFIGS["c3"]
    N = cfg["grid"]
    rp, ci, va = convdiff3d(N, (cfg["beta"],) * 3)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    A.device_arrays()
    n = A.n
    b_host = rhs_gaussian(n, 0)
    b = torch.from_numpy(b_host).cuda()
    th = sg.make_sketch(sg.SketchKind.PSRHT, cfg["k"], n, 0)
    th.device_data()
    solve = lambda pol, rhs, lagged=False: sg.gmres_restarted(  # noqa: E731
        A, rhs, th, pol, cfg["restart"], cfg["max_iters"], cfg["tol"], lagged=lagged)
    out = {}
    clocks = Clocks(0)
    # standard RGS-Arnoldi (the reference's algorithm) for both bases, then the
    # one-synchronisation variant as "<basis>_lagged".  One
    # untimed pass over all four first, so the first timed variant does not
    # absorb the GPU's clock/power ramp (measured: fp64 standard 1849-2106
    # steps/s across boxes when timed first, the others stable)
    variants = ("f64", "mixed", "f64_lagged", "mixed_lagged")
    for pname in variants:
        solve(sg.policy_from_name(pname.split("_")[0]), b, pname.endswith("_lagged"))
    for pname in variants:
        pol = sg.policy_from_name(pname.split("_")[0])
        lag = pname.endswith("_lagged")
        for _ in range(args.warmup):
            solve(pol, b, lag)
        torch.cuda.synchronize()
        lc0 = _lib.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        its = 0
        for _ in range(args.steps):
            res = solve(pol, b, lag)
            its += res.iterations
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out[pname] = {"steps_per_s": its / (ms / 1e3), "iterations": res.iterations,
                      "cycles": res.cycles, "relres": res.final_residual,
                      "ms_per_solve": ms / args.steps,
                      "gpu_launches": _lib.launch_count() - lc0}
    clk = clocks.stop()

    # roofline of the dominant kernel (fused column kernel) over one fp64 solve
    evs = []
    orig = gsm.RgsState._column

    def timed_column(self, i, w_ptr, w_code, normalize_prev, sketch, **kw):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        r = orig(self, i, w_ptr, w_code, normalize_prev, sketch, **kw)
        b_.record()
        evs.append((i, a_, b_))
        return r

    gsm.RgsState._column = timed_column
    try:
        solve(sg.UNIFIED64, b)
    finally:
        gsm.RgsState._column = orig
    torch.cuda.synchronize()
    tot_ms = sum(a_.elapsed_time(b_) for _, a_, b_ in evs)
    tot_b = sum(update_alg_bytes(n, i, 8, 8) for i, _, _ in evs)
    peak, peak_kind = _peaks()
    ach = tot_b / (tot_ms / 1e3) / 1e9
    f64_ms = out["f64"]["ms_per_solve"]
    roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
            "frac": round(ach / peak, 4), "frac_nominal_8tbs": round(ach / 8000.0, 4),
            "traffic": _traffic("c3")[0], "traffic_note": _traffic("c3")[1],
            "kernel": "rgs_column_kernel (Q stream + SRHT epilogue), fp64 basis",
            "peak_source": peak_kind, "share_of_step": round(tot_ms / f64_ms, 4),
            "launches": len(evs), "avg_launch_us": round(1e3 * tot_ms / len(evs), 2),
            "note": "algorithmic bytes include w = A q / alpha, which the SpMV has just "
                    "written and the column kernel reads from L2, and early columns' Q "
                    "slices that fit in L2; so achieved/peak can exceed 1"}

    # e2e: numpy b in, numpy x out through the public call (fp64 basis)
    e2e = None
    if not args.no_e2e:
        solve(sg.UNIFIED64, b_host)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ne = max(1, min(args.steps, 3))
        its = 0
        for _ in range(ne):
            r = solve(sg.UNIFIED64, b_host)
            its += r.iterations
        dt = time.perf_counter() - t0
        e2e = {"value": its / dt, "unit": "steps/s", "h2d_bytes_per_step": n * 8,
               "d2h_bytes_per_step": n * 8, "ms_per_step": 1e3 * dt / ne,
               "path": "gmres_restarted(numpy b) -> numpy x"}
    cpu = None
    if not args.no_cpu:
        threads = os.cpu_count() or 1
        v, dt = cpu_gmres_sample(40, threads)
        cpu = {"value": v, "unit": "steps/s", "cores": threads, "kind": "port",
               "sample": f"40 Arnoldi steps of c3 at full size (n={n}, k={cfg['k']}, fp64), "
                         f"oracle port, {dt:.1f} s"}
    print(json.dumps({"metric": "RGMRES Arnoldi steps/s", "value": out["f64"]["steps_per_s"],
                      "unit": "steps/s", "n_gpus": 1, "steps": args.steps,
                      "warmup": args.warmup, "ms_per_step": f64_ms,
                      "higher_is_better": True, "scaling": "weak",
                      "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": "c3", **cfg,
                                 "l2": "inputs larger than L2 (basis, CSR >> 126 MB)"},
                      "results": out, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                      "gpu_launches": out["f64"]["gpu_launches"], "clocks": clk}), flush=True)


def run_gmres_sharded(args, comm):
    """c3 at N > 1: row-sharded restarted RGMRES (strong scaling over n = 2^21
    rows); steps/s of the whole job, device time as the max over ranks."""
    import torch
    import paper_2011_05090_b200 as sg
    from paper_2011_05090_b200 import _lib
    from paper_2011_05090_b200.workloads import CONFIGS, convdiff3d, rhs_gaussian
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    cfg = CONFIGS["c3"]
    N = cfg["grid"]
    rp, ci, va = convdiff3d(N, (cfg["beta"],) * 3)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    b = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
    th = sg.make_sketch(sg.SketchKind.PSRHT, cfg["k"], A.n, 0)
    th.device_data()
    out = {}
    clocks = Clocks(local)
    # standard RGS-Arnoldi, then the one-synchronisation variant (one [s'; p']
    # all-reduce per step instead of two k-vector all-reduces)
    for pname in ("f64", "mixed", "f64_lagged", "mixed_lagged"):
        pol = sg.policy_from_name(pname.split("_")[0])
        lag = pname.endswith("_lagged")
        solve = lambda: sg.gmres_restarted(A, b, th, pol, cfg["restart"],  # noqa: E731
                                           cfg["max_iters"], cfg["tol"], comm=comm,
                                           lagged=lag)
        for _ in range(args.warmup):
            solve()
        torch.cuda.synchronize()
        torch.distributed.barrier()
        lc0 = _lib.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        its = 0
        for _ in range(args.steps):
            res = solve()
            its += res.iterations
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(ms, op=torch.distributed.ReduceOp.MAX)
        ms = float(ms)
        out[pname] = {"steps_per_s": its / (ms / 1e3), "iterations": res.iterations,
                      "cycles": res.cycles, "relres": res.final_residual,
                      "ms_per_solve": ms / args.steps,
                      "gpu_launches": _lib.launch_count() - lc0}
    clk = clocks.stop()
    if comm.rank == 0:
        print(json.dumps({"metric": "RGMRES Arnoldi steps/s", "value": out["f64"]["steps_per_s"],
                          "unit": "steps/s", "n_gpus": comm.world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": out["f64"]["ms_per_solve"],
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                          "dtype": "f64", "data": "synthetic",
                          "config": {"workload": "c3", **cfg,
                                     "parallelism": f"row-shard x{comm.world}"},
                          "results": out, "gpu_launches": out["f64"]["gpu_launches"],
                          "clocks": clk}), flush=True)
    torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None,
                    help="c0|c0r|c1|c2|c3|c4; default c1 at N = 1, c2 (strong) at N > 1")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="N > 1 on c1: weak (1e6 rows per GPU, default) or strong (n = 1e6 split)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--columns", type=int, default=None,
                    help="override the config's column count (functional runs; the workload "
                         "name records it)")
    ap.add_argument("--cpu-cols", type=int, default=96,
                    help="columns of the CPU baseline sample (about 10-30 s of host work at c1)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="N >= 4: skip the c4 line")
    ap.add_argument("--no-c2", action="store_true",
                    help="default N = 1 run: skip the c2 strong-scaling point (results.c2_strong_n1)")
    args = ap.parse_args()
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    defaulted = args.config is None
    if args.config is None:
        # N = 1: BASELINE configs[1] (the metric's config); N > 1: configs[2],
        # the row-sharded c2, strong-scaled with the same Theta at every N
        args.config = "c2" if max(world_env, args.gpus) > 1 else "c1"
    if args.impl == "reference":
        run_reference(args, args.config)
        return
    if args.config == "c3":
        run_gmres(args)
        return
    from paper_2011_05090_b200.distributed import init_from_env
    # SGS_DIST_BACKEND=gloo runs several ranks on one GPU: a functional check of
    # the sharded path only, never a timing
    comm = init_from_env(os.environ.get("SGS_DIST_BACKEND", "nccl"))
    line = run_qr(args, args.config, comm)
    world = comm.world if comm else 1
    if args.config == "c2" and world >= 4 and not args.no_c4 and args.columns is None:
        # BASELINE configs[4] exists only at 4 and 8 GPUs: its line rides along
        # with c2's (fewer timed steps; W and Q are 201 GB each)
        import copy
        import torch
        torch.cuda.empty_cache()
        a4 = copy.copy(args)
        a4.steps, a4.warmup, a4.no_e2e, a4.no_cpu = min(args.steps, 3), min(args.warmup, 3), True, True
        l4 = run_qr(a4, "c4", comm)
        if line is not None and l4 is not None:
            line["results"] = {"c4": {k_: l4.get(k_) for k_ in (
                "value", "unit", "ms_per_step", "steps", "warmup", "config", "hbm_gbs_whole_step",
                "hbm_frac_whole_step", "roofline", "gpu_launches", "graph", "unavailable")}}
    if (defaulted and world == 1 and not args.no_c2 and args.columns is None
            and line is not None):
        # the N = 1 point of the c2 strong-scaling curve that the N > 1 runs
        # print (their default): same workload, same Theta, one GPU (W and Q
        # are 67 GB each); fewer timed steps, no e2e / CPU legs
        import copy
        import torch
        torch.cuda.empty_cache()
        a2 = copy.copy(args)
        a2.steps, a2.warmup, a2.no_e2e, a2.no_cpu = min(args.steps, 2), 1, True, True
        try:
            l2 = run_qr(a2, "c2", None)
        except Exception as e:  # the c1 line stands on its own
            l2 = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
        if l2 is not None:
            line["results"] = {"c2_strong_n1": {k_: l2.get(k_) for k_ in (
                "value", "unit", "ms_per_step", "steps", "warmup", "config",
                "hbm_gbs_whole_step", "hbm_frac_whole_step", "roofline", "gpu_launches", "graph",
                "clocks", "unavailable") if k_ in l2}}
    if line is not None:
        print(json.dumps(line), flush=True)
    if comm:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
