"""The fused SpMV + SRHT launch of the Arnoldi step (sgs_csr_spmv_srht): w = A q
and the partials of Theta w must equal the plain SpMV followed by the
stand-alone sketch bit for bit (reference: w = A v, krylov.py:81-83 and
gram_schmidt.py:297 sketching it through sketch.py:90-109)."""

import numpy as np
import pytest
import torch

import paper_2011_05090_b200 as sg
from paper_2011_05090_b200 import _lib
from paper_2011_05090_b200.workloads import convdiff3d

pytestmark = pytest.mark.gpu


def _scratch(n, k, dev):
    lib = _lib.load()
    tv = torch.empty(int(lib.sgs_spmv_srht_tilevec_elems(n, k)), dtype=torch.float64, device=dev)
    cnt = torch.zeros(int(lib.sgs_spmv_srht_counter_elems(n)), dtype=torch.int64, device=dev)
    return tv, cnt


def _fused(A, th, x, alpha, y, parts, tv, cnt, st, row0=0, rp=None):
    d = th.device_data(y.device)
    if rp is None:
        rp, ci, va = A.device_arrays(y.device)
        n = A.n
    else:
        rp, ci, va, n = rp
    _lib.call("sgs_csr_spmv_srht", n, rp.data_ptr(), ci.data_ptr(), va.data_ptr(), x.data_ptr(),
              _lib.dtype_code(x.dtype), None, alpha.data_ptr() if alpha is not None else None,
              y.data_ptr(), row0, th.log2_block, d["bits"].data_ptr() + (row0 // 32) * 4,
              d["samples"].data_ptr(), th.k, tv.data_ptr(), cnt.data_ptr(), parts.data_ptr(),
              st.ptr, _lib.stream_ptr())


@pytest.mark.parametrize("N,kind,k,dt", [(128, "psrht", 600, torch.float64),
                                         (128, "psrht", 600, torch.float32),
                                         (20, "psrht", 200, torch.float64),
                                         (32, "block_srht", 1500, torch.float64),
                                         (24, "psrht", 2048, torch.float32)])
def test_fused_spmv_srht_equals_spmv_then_sketch(cuda, N, kind, k, dt):
    """c3's 128^3 operator (512 tiles, groups of 8), a ragged n = 8000 (a
    partial last tile), a block-SRHT with 4096-row blocks, k up to 2048;
    fp64 and fp32 basis columns, with the 1/alpha scaling.  Three launches in
    a row reuse the monotonic counters."""
    rp, ci, va = convdiff3d(N)
    n = N ** 3
    A = sg.SparseMatrix(n=n, row_ptr=rp, col_idx=ci, values=va)
    kw = {"block_log2": 12} if kind == "block_srht" else {}
    th = sg.make_sketch(sg.SketchKind(kind), k, n, 3, **kw)
    g = torch.Generator(device="cuda").manual_seed(11)
    alpha = torch.tensor([3.25], dtype=torch.float64, device=cuda)
    st = _lib.Status(cuda)
    tv, cnt = _scratch(n, k, cuda)
    npart = th.nparts(n)
    for rep in range(3):
        x = torch.randn(n, dtype=torch.float64, device=cuda, generator=g).to(dt)
        y0 = torch.empty(n, dtype=torch.float64, device=cuda)
        y1 = torch.empty_like(y0)
        p0 = torch.empty((npart, k), dtype=torch.float64, device=cuda)
        p1 = torch.full_like(p0, float("nan"))
        A.spmv_into(x.data_ptr(), _lib.dtype_code(dt), y0, alpha=alpha, status=st)
        th.partials_into(y0, _lib.SGS_F64, n, 1, p0, status=st)
        _fused(A, th, x, alpha, y1, p1, tv, cnt, st)
        torch.cuda.synchronize()
        assert torch.equal(y0, y1), rep
        assert torch.equal(p0, p1), rep
    # the sketch itself: sum of the partials (scaled) is Theta w
    ref = th.apply(y1)
    got = p1.sum(0) * th.scale
    assert torch.allclose(got, ref, rtol=1e-12, atol=1e-12 * float(ref.abs().max()))


def test_fused_spmv_srht_stopped_launch_keeps_counters(cuda):
    """A launch that finds the status block stopped writes nothing but still
    counts, so the next launch after a reset completes every tile and group."""
    N, k = 32, 300
    rp, ci, va = convdiff3d(N)
    n = N ** 3
    A = sg.SparseMatrix(n=n, row_ptr=rp, col_idx=ci, values=va)
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 5)
    st = _lib.Status(cuda)
    tv, cnt = _scratch(n, k, cuda)
    x = torch.randn(n, dtype=torch.float64, device=cuda)
    y = torch.full((n,), 7.0, dtype=torch.float64, device=cuda)
    p = torch.full((th.nparts(n), k), 7.0, dtype=torch.float64, device=cuda)
    st.buf[0] = 2  # a recorded outcome: kernels return at once
    _fused(A, th, x, None, y, p, tv, cnt, st)
    torch.cuda.synchronize()
    assert bool((y == 7.0).all()) and bool((p == 7.0).all())
    st.clear_code()
    _fused(A, th, x, None, y, p, tv, cnt, st)
    y0 = torch.empty_like(y)
    p0 = torch.empty_like(p)
    A.spmv_into(x.data_ptr(), _lib.SGS_F64, y0, status=st)
    th.partials_into(y0, _lib.SGS_F64, n, 1, p0, status=st)
    torch.cuda.synchronize()
    assert torch.equal(y, y0) and torch.equal(p, p0)


def test_fused_spmv_srht_row_shard(cuda):
    """A row shard (row0 = 2 tiles) of a block-SRHT: the shard's rows of the
    operator (column indices relative to a halo window starting at col0) and
    the shard's sign words / blocks, as the sharded RGMRES uses it."""
    from paper_2011_05090_b200.krylov import _RowBlock
    N, k = 32, 400
    rp, ci, va = convdiff3d(N)
    n = N ** 3
    A = sg.SparseMatrix(n=n, row_ptr=rp, col_idx=ci, values=va)
    th = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, k, n, 9, block_log2=13)
    row0, nrows = 2 * 4096, 3 * 4096 + 1000
    col0 = row0 - N * N
    blk = _RowBlock(A, row0, nrows, cuda, col0=col0)
    xg = torch.randn(n, dtype=torch.float64, device=cuda)
    xw = xg[col0:].contiguous()
    st = _lib.Status(cuda)
    tv, cnt = _scratch(nrows, k, cuda)
    npart = th.nparts(nrows)
    y0 = torch.empty(nrows, dtype=torch.float64, device=cuda)
    y1 = torch.empty_like(y0)
    p0 = torch.empty((npart, k), dtype=torch.float64, device=cuda)
    p1 = torch.empty_like(p0)
    blk.spmv_into(xw.data_ptr(), _lib.SGS_F64, y0, status=st)
    th.partials_into(y0, _lib.SGS_F64, nrows, 1, p0, n_local=nrows, row0=row0, status=st)
    _fused(None, th, xw, None, y1, p1, tv, cnt, st, row0=row0,
           rp=(blk.rp, blk.ci, blk.va, nrows))
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    assert torch.equal(p0, p1)
    # and the rows are the operator's
    ref = A.matvec(xg.cpu().numpy())[row0:row0 + nrows]
    assert np.allclose(y1.cpu().numpy(), ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("policy,lagged", [("f64", False), ("mixed", False), ("f64", True),
                                           ("mixed", True)])
def test_gmres_fused_and_unfused_spmv_sketch_agree(cuda, policy, lagged, monkeypatch):
    """RGMRES with the fused SpMV + SRHT and with two launches
    (SGS_SPMV_SRHT=0): identical iterations and solution bits."""
    from paper_2011_05090_b200 import krylov as kr
    from paper_2011_05090_b200.workloads import rhs_gaussian
    N = 24
    rp, ci, va = convdiff3d(N)
    A = sg.SparseMatrix(n=N ** 3, row_ptr=rp, col_idx=ci, values=va)
    b = rhs_gaussian(A.n, 0)
    th = sg.make_sketch(sg.SketchKind.PSRHT, 240, A.n, 0)
    pol = sg.policy_from_name(policy)
    out = []
    for fused in (True, False):
        monkeypatch.setattr(kr, "_SPMV_SRHT", fused)
        r = sg.gmres(A, b, m=80, theta=th, policy=pol, tol=1e-8, lagged=lagged)
        out.append(r)
    assert out[0].iterations == out[1].iterations
    assert np.array_equal(np.asarray(out[0].x), np.asarray(out[1].x))
