"""Row-sharded RGS on two CPU ranks (gloo): the host logic of the multi-GPU
path.  Each rank owns a tile-aligned row range (workloads.shard_rows), runs
the n-dimensional steps on its rows, and gets every sketch as the all-reduce
of its local (zero-padded) sketch; the k-dimensional least squares is
replicated.  The result must equal the unsharded oracle: this is the
structure RgsState(comm=...) runs on the GPUs with NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import OracleSketch, oracle_rgs_factorize
from oracle.ref_rgs import householder_lsq
from paper_2011_05090_b200.distributed import TorchComm
from paper_2011_05090_b200.workloads import make_w, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sharded_rgs(W, op, comm, row0, n_loc):
    """RGS with sharded rows (fp64): local update, all-reduced sketches."""
    n, m = W.shape
    k = op.k

    def sketch(local):
        full = np.zeros(n)
        full[row0:row0 + n_loc] = local
        t = torch.from_numpy(op.apply(full))  # linear: sum of per-rank sketches
        comm.allreduce_(t)
        return t.numpy()

    ls = householder_lsq(k, np.float64)
    Q = np.zeros((n_loc, m))
    R = np.zeros((m, m))
    S = np.zeros((k, m))
    for i in range(m):
        w = W[row0:row0 + n_loc, i]
        p = sketch(w)
        if i == 0:
            qp, sp, r = w.copy(), p.copy(), np.zeros(0)
        else:
            r = ls.solve(p)
            qp = w - Q[:, :i] @ r
            sp = sketch(qp)
        rii = float(np.sqrt(np.sum(sp * sp)))
        S[:, i] = sp / rii
        Q[:, i] = qp / rii
        R[:i, i] = r
        R[i, i] = rii
        ls.add(S[:, i])
    return Q, R, S


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = TorchComm()
    # 1. the all-reduce hook
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    comm.allreduce_(t)
    assert float(t) == sum(range(1, world + 1))
    # 2. sharded RGS on a tile-aligned row partition
    n, m, k = 3 * 4096 + 123, 12, 64
    W = make_w(n, m, 1e-4, 2)
    op = OracleSketch("psrht", k, n, 2)
    row0, n_loc = shard_rows(n, world, rank, 4096)
    Q, R, S = _sharded_rgs(W, op, comm, row0, n_loc)
    out[rank] = (row0, n_loc, Q, R, S)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_rgs_matches_unsharded():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    n, m, k = 3 * 4096 + 123, 12, 64
    W = make_w(n, m, 1e-4, 2)
    ref = oracle_rgs_factorize(W, OracleSketch("psrht", k, n, 2), "f64")
    Q = np.concatenate([out[r][2] for r in range(world)], axis=0)
    assert [out[r][0] for r in range(world)] == [0, 8192]
    for r in range(world):  # replicated k-dimensional state is identical
        assert np.array_equal(out[r][3], out[0][3])
        assert np.array_equal(out[r][4], out[0][4])
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(Q, ref["Q"]) < 1e-12
    assert rel(out[0][3], ref["R"]) < 1e-12
    assert rel(out[0][4], ref["S"]) < 1e-12


class _StubBlock:
    """Stands in for the device row block (the halo test moves vectors only)."""

    def __init__(self, *a, **kw):
        pass


def _halo_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # a subgroup that excludes global rank 0: group ranks 0, 1, 2 are global
    # ranks 1, 2, 3, so a peer passed as a global rank would reach the wrong
    # process (advisor finding on krylov.py's halo P2POps)
    grp = dist.new_group([1, 2, 3])
    if rank != 0:
        from paper_2011_05090_b200 import krylov
        krylov._RowBlock = _StubBlock
        n = 6144
        # 1-D three-point stencil: each shard's rows touch one row of each neighbour
        rp = np.zeros(n + 1, dtype=np.int64)
        cols = []
        for i in range(n):
            row = [j for j in (i - 1, i, i + 1) if 0 <= j < n]
            cols += row
            rp[i + 1] = len(cols)
        A = krylov.SparseMatrix(n=n, row_ptr=rp, col_idx=np.asarray(cols, dtype=np.int64),
                                values=np.ones(len(cols)))
        comm = TorchComm(grp)
        d = krylov._Dist(comm, A, 1024, "cpu")
        x = torch.arange(n, dtype=torch.float64) * 0.5 + 1.0
        buf, _ = d.window(x[d.row0:d.row0 + d.n_loc].clone())
        full = d.full(x[d.row0:d.row0 + d.n_loc].clone())
        out[rank] = (d.halo, d.wlo, d.whi, buf.numpy().copy(),
                     bool(torch.equal(full, x)), comm.rank)
    dist.barrier()
    dist.destroy_process_group()


def test_halo_exchange_in_a_subgroup():
    world = 4
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_halo_worker, args=(world, port, out), nprocs=world, join=True)
    x = np.arange(6144, dtype=np.float64) * 0.5 + 1.0
    for g in (1, 2, 3):
        halo, wlo, whi, buf, full_ok, grank = out[g]
        assert grank == g - 1
        assert halo, "the 3-point stencil's windows are narrow: halo path expected"
        assert np.array_equal(buf, x[wlo:whi]), g
        assert full_ok
    assert (out[1][1], out[1][2]) == (0, 2049)
    assert (out[2][1], out[2][2]) == (2047, 4097)


class _FakePeerLib:
    """sgs_peer_* stand-ins that succeed (a rank whose IPC set-up works)."""

    def __init__(self):
        self.freed = []

    def sgs_peer_bytes(self, world, k, cl):
        return 4096

    def sgs_peer_alloc(self, nbytes, out):
        out._obj.value = 0x1000
        return 0

    def sgs_peer_export(self, area, buf):
        buf.raw = b"h" * 64
        return 0

    def sgs_peer_import(self, buf, out):
        out._obj.value = 0x2000
        return 0

    def sgs_peer_desc_create(self, world, rank, k, areas, out):
        out._obj.value = 0x3000
        return 0

    def sgs_peer_desc_free(self, d):
        self.freed.append("desc")
        return 0

    def sgs_peer_unimport(self, p):
        self.freed.append("import")
        return 0

    def sgs_peer_free(self, p):
        self.freed.append("area")
        return 0


def _peer_worker(rank, world, port, out, fake_ranks):
    import warnings
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2011_05090_b200 import _lib
    from paper_2011_05090_b200.distributed import PeerExchange
    fake = _FakePeerLib()
    if rank in fake_ranks:
        _lib.load = lambda: fake
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        ex = PeerExchange.get(TorchComm(), 64, 16)
        again = PeerExchange.get(TorchComm(), 64, 16)  # cached outcome, no collective
    out[rank] = (ex is None, again is None, [str(w.message) for w in caught],
                 None if ex is None else (ex.ok, ex.desc), fake.freed)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("fake_ranks", [(), (1,), (0, 1)])
def test_peer_exchange_setup_is_agreed_across_ranks(fake_ranks):
    """The peer-memory exchange is set up collectively: a rank whose
    allocation, export or import fails still joins the host collectives, and
    the ranks agree (MIN of their outcomes) - all use the exchange or all fall
    back to the NCCL all-reduce, never a mix that would leave one rank
    spinning on flags the others never write.  Here the real library fails
    without a GPU; fake_ranks succeed through stand-ins."""
    world = 2
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_peer_worker, args=(world, port, out, fake_ranks), nprocs=world, join=True)
    if len(fake_ranks) == world:
        for r in range(world):
            none, again, warns, state, freed = out[r]
            assert not none and not again and state == (True, 0x3000) and not warns
    else:
        for r in range(world):
            none, again, warns, state, freed = out[r]
            assert none and again
            assert any("peer-memory exchange unavailable" in w for w in warns)
            if r in fake_ranks:  # its own area is freed; it never imported the
                assert freed == ["area"]  # failed rank's (missing) handle
