"""The sharded RGS path under a collective with NCCL's stream semantics, on
one GPU.

NCCL cannot run two ranks on one GPU, so two checks stand in for it:

* ``SideStreamComm`` is a one-rank communicator that behaves like
  ProcessGroupNCCL on the device: the collective runs on its own stream,
  ordered by events against the caller's stream.  To make an ordering bug
  visible, the tensor is zeroed on the caller's stream and the true values
  are written back only on the side stream, after a spin delay.  Any kernel
  that read the k-vector before waiting for the side stream - in particular
  the PDL-launched LS step behind the event wait - would see zeros, and the
  factors would differ from the unsharded run.
* A real NCCL process group of world size 1 (spawned process): the NCCL
  collective code paths, eager and captured in a CUDA graph, must reproduce
  the unsharded factorisation bit for bit - with s' summed by the LS
  launch's peer-memory exchange (CUDA IPC areas, release/acquire flags at
  system scope; here the one rank is its own peer) and with the per-column
  NCCL all-reduce (SGS_PEER=0).  With two or more GPUs a 2-rank
  NCCL run is checked against the gloo run (skipped on one GPU).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2011_05090_b200 as sg
from paper_2011_05090_b200.workloads import make_w

pytestmark = pytest.mark.gpu


class SideStreamComm:
    rank, world, group, capturable = 0, 1, None, True

    def __init__(self, delay_cycles: int = 200_000):
        self.side = torch.cuda.Stream()
        self.delay = delay_cycles
        self.saved = {}
        self.calls = 0

    def allreduce_(self, t: torch.Tensor) -> None:
        key = (t.numel(), t.dtype)
        buf = self.saved.get(key)
        if buf is None:
            buf = self.saved[key] = torch.empty(t.numel(), dtype=t.dtype, device=t.device)
        cur = torch.cuda.current_stream()
        buf.copy_(t.reshape(-1))
        t.zero_()                         # what a consumer sees if it does not wait
        self.side.wait_stream(cur)
        with torch.cuda.stream(self.side):
            torch.cuda._sleep(self.delay)
            t.reshape(-1).copy_(buf)      # the "reduced" result lands late
        cur.wait_stream(self.side)
        self.calls += 1


def _factor(W, th, pol, comm=None, graph=False):
    n, m = W.shape
    Wd = torch.from_numpy(np.ascontiguousarray(W.T)).cuda()   # (m, n) column-major W
    kw = {"comm": comm, "row0": 0, "n_local": n} if comm is not None else {}
    st = sg.RgsState(th, pol, capacity=m + 1, breakdown_factor=0.0, **kw)
    if graph:
        g = st.capture_factorization(Wd, n, m)
        for _ in range(2):    # replays re-run every kernel and collective
            g.replay()
        st.finish()
    else:
        st.factorize_columns(Wd, n, m)
    f = st.device_factors()
    return [t.cpu().numpy() for t in (f.Q, f.R, f.S, f.P)]


CASES = [("psrht", "mixed", 3 * 4096 + 777, 40, 200), ("block_srht", "f64", 4 * 4096, 30, 160),
         ("gaussian", "f64", 5003, 24, 96)]


@pytest.mark.parametrize("kind,pol,n,m,k", CASES)
@pytest.mark.parametrize("graph", [False, True])
def test_side_stream_collective_ordering(cuda, kind, pol, n, m, k, graph):
    kw = {"block_log2": 12} if kind == "block_srht" else {}
    th = sg.make_sketch(sg.SketchKind(kind), k, n, 3, **kw)
    W = make_w(n, m, 1e-6, 3, dtype=np.float32 if pol == "mixed" else np.float64)
    P = sg.policy_from_name(pol)
    ref = _factor(W, th, P)
    comm = SideStreamComm()
    if graph:
        _factor(W, th, P, comm)   # allocate the comm's buffers before capturing
    got = _factor(W, th, P, comm, graph=graph)
    assert comm.calls >= m  # one k-vector per column (+ the P batch)
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(rank, world, port, backend, out):
    import torch.distributed as dist
    from paper_2011_05090_b200.distributed import TorchComm
    from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian, shard_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group(backend, rank=rank, world_size=world)
    comm = TorchComm()
    n, m, k = 3 * 4096 + 777, 40, 200
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 3)
    row0, n_loc = shard_rows(n, world, rank, th.row_align())
    W = make_w(n, m, 1e-6, 3, dtype=np.float32)[row0:row0 + n_loc]
    Wd = torch.from_numpy(np.ascontiguousarray(W.T)).cuda()
    res = {}
    for graph in (False, True):
        st = sg.RgsState(th, sg.MIXED32_64, capacity=m + 1, breakdown_factor=0.0, comm=comm,
                         row0=row0, n_local=n_loc)
        if graph and comm.capturable:
            st.factorize_columns(Wd, n_loc, m)  # communicator warm
            st.m = 0
            g = st.capture_factorization(Wd, n_loc, m)
            g.replay()
            st.finish()
        elif graph:
            continue
        else:
            st.factorize_columns(Wd, n_loc, m)
        f = st.device_factors()
        res[graph] = tuple(t.cpu().numpy() for t in (f.Q, f.R, f.S, f.P))
        if comm.capturable:  # NCCL: s' summed by the peer-memory exchange in the LS launch
            assert st.__dict__.get("_peer") is not None
    if comm.capturable:  # and with the per-column NCCL all-reduce instead (SGS_PEER=0)
        from paper_2011_05090_b200 import gram_schmidt as gsm
        old, gsm._PEER = gsm._PEER, False
        try:
            st = sg.RgsState(th, sg.MIXED32_64, capacity=m + 1, breakdown_factor=0.0, comm=comm,
                             row0=row0, n_local=n_loc)
            st.factorize_columns(Wd, n_loc, m)
            assert st.__dict__.get("_peer") is None
            f = st.device_factors()
            res["nccl_allreduce"] = tuple(t.cpu().numpy() for t in (f.Q, f.R, f.S, f.P))
        finally:
            gsm._PEER = old
    # the end-to-end path (pinned host W, chunked H2D / compute / D2H) sharded
    pin = torch.empty((m, n_loc), dtype=torch.float32, pin_memory=True)
    pin.copy_(torch.from_numpy(np.ascontiguousarray(W.T)))
    f, _ = sg.rgs_factorize(pin.numpy().T, th, sg.MIXED32_64, breakdown_factor=0.0, comm=comm,
                            row0=row0, with_certificate=False)
    res["pipelined"] = tuple(np.asarray(x) for x in (f.Q, f.R, f.S, f.P))
    # row-sharded RGMRES: halo exchange / all-gather over this backend
    N = 12
    rp, ci, va = convdiff3d(N)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    b = torch.from_numpy(rhs_gaussian(A.n, 0)).cuda()
    th2 = sg.make_sketch(sg.SketchKind.PSRHT, 120, A.n, 0)
    g = sg.gmres(A, b, m=60, theta=th2, policy=sg.UNIFIED64, tol=1e-8, comm=comm)
    x = g.x.cpu().numpy() if isinstance(g.x, torch.Tensor) else np.asarray(g.x)
    out[rank] = (row0, n_loc, res, g.iterations, x)
    dist.barrier()
    dist.destroy_process_group()


def _spawn(world, backend):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_nccl_worker, args=(world, _free_port(), backend, out), nprocs=world, join=True)
    return dict(out)


def test_nccl_world1_eager_and_graph_match_unsharded(cuda):
    out = _spawn(1, "nccl")
    row0, n_loc, res, its, x = out[0]
    n, m, k = 3 * 4096 + 777, 40, 200
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 3)
    ref = _factor(make_w(n, m, 1e-6, 3, dtype=np.float32), th, sg.MIXED32_64)
    for variant in (False, True, "nccl_allreduce", "pipelined"):  # peer eager/graph, NCCL, e2e
        for a, b in zip(ref, res[variant]):
            assert np.array_equal(a, b), variant
    from paper_2011_05090_b200.workloads import convdiff3d, rhs_gaussian
    N = 12
    rp, ci, va = convdiff3d(N)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    th2 = sg.make_sketch(sg.SketchKind.PSRHT, 120, A.n, 0)
    r = sg.gmres(A, rhs_gaussian(A.n, 0), m=60, theta=th2, policy=sg.UNIFIED64, tol=1e-8)
    assert its == r.iterations
    assert np.linalg.norm(x - r.x) <= 1e-12 * np.linalg.norm(r.x)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="a 2-rank NCCL run needs 2 GPUs")
def test_nccl_two_ranks_match_gloo(cuda):
    a = _spawn(2, "nccl")
    b = _spawn(2, "gloo")
    for r in range(2):
        for x, y in zip(a[r][2][False], b[r][2][False]):
            assert np.array_equal(x, y)
        for x, y in zip(a[r][2][True], a[r][2][False]):
            assert np.array_equal(x, y)
        assert a[r][3] == b[r][3]
        assert np.array_equal(a[r][4], b[r][4])
