"""The row-sharded RGS path (RgsState(comm=...)) on two ranks sharing cuda:0.

The collective is gloo on CUDA tensors (host-staged), so no kernel waits on
another process; the sharded kernels (row offsets into the sign bitmask and
the block structure, local partial reduction, all-reduce, replicated
k-dimensional state) are the ones the NCCL multi-GPU run executes."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    "psrht_mixed": dict(kind="psrht", n=3 * 4096 * 4 + 1000, m=40, k=200, pol="mixed", blog=None),
    "block_f64": dict(kind="block_srht", n=4 * 8192, m=30, k=160, pol="f64", blog=13),
    # device-generated Rademacher signs: the shard reads its rows of the packed
    # sign array (row0 need not be tile-aligned for the dense chunking)
    "rademacher_f64": dict(kind="rademacher", n=6001, m=24, k=120, pol="f64", blog=None),
    "gaussian_mixed": dict(kind="gaussian", n=7003, m=20, k=100, pol="mixed", blog=None),
}


def _worker(rank, world, port, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2011_05090_b200 as sg
    from paper_2011_05090_b200.distributed import TorchComm
    from paper_2011_05090_b200.workloads import make_w, shard_rows
    c = CASES[case]
    kw = {"block_log2": c["blog"]} if c["blog"] else {}
    th = sg.make_sketch(sg.SketchKind(c["kind"]), c["k"], c["n"], 4, **kw)
    comm = TorchComm()
    row0, n_loc = shard_rows(c["n"], world, rank, th.row_align())
    dt = np.float32 if c["pol"] == "mixed" else np.float64
    W = make_w(c["n"], c["m"], 1e-6, 4, dtype=dt)[row0:row0 + n_loc]
    f, _ = sg.rgs_factorize(np.asfortranarray(W), th, sg.policy_from_name(c["pol"]),
                            breakdown_factor=0.0, comm=comm, row0=row0, with_certificate=False)
    # the pinned host shard takes the overlapped H2D/compute/D2H pipeline, which
    # all-reduces P chunk by chunk: same kernels and order, so the same bits
    pin = torch.empty((c["m"], n_loc), dtype=torch.from_numpy(W[:1]).dtype, pin_memory=True)
    pin.copy_(torch.from_numpy(np.ascontiguousarray(W.T)))
    fp, _ = sg.rgs_factorize(pin.numpy().T, th, sg.policy_from_name(c["pol"]),
                             breakdown_factor=0.0, comm=comm, row0=row0, with_certificate=False)
    for a, b in ((f.Q, fp.Q), (f.R, fp.R), (f.S, fp.S), (f.P, fp.P)):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    out[rank] = (row0, n_loc, f.Q, f.R, f.S, f.P)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", list(CASES))
def test_two_rank_sharded_factorization(cuda, case):
    import paper_2011_05090_b200 as sg
    from oracle import factor_metrics, rel_diff
    from paper_2011_05090_b200.workloads import make_w
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    c = CASES[case]
    kw = {"block_log2": c["blog"]} if c["blog"] else {}
    th = sg.make_sketch(sg.SketchKind(c["kind"]), c["k"], c["n"], 4, **kw)
    dt = np.float32 if c["pol"] == "mixed" else np.float64
    W = make_w(c["n"], c["m"], 1e-6, 4, dtype=dt)
    ref, _ = sg.rgs_factorize(W, th, sg.policy_from_name(c["pol"]), breakdown_factor=0.0)
    Q = np.concatenate([out[r][2] for r in range(world)], axis=0)
    for r in range(world):  # the replicated k-dimensional state is bit-identical
        for j in (3, 4, 5):
            assert np.array_equal(out[r][j], out[0][j])
    R, S = out[0][3], out[0][4]
    if c["pol"] == "f64":
        assert rel_diff(Q, ref.Q) < 1e-10 and rel_diff(R, ref.R) < 1e-10
    ours = factor_metrics(W, Q, R, S)
    theirs = factor_metrics(W, ref.Q, ref.R, ref.S)
    for key in ours:
        assert ours[key] <= 10 * max(theirs[key], 1e-15), (key, ours[key], theirs[key])
