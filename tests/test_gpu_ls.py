"""The sketched least-squares kernel on its own (sgs_ls_step through
sketched_lsq), ported from the reference's tests/test_gram_schmidt.py:96-114:
the solver against numpy's lstsq on near-orthonormal S, and the rank-deficient
sketched basis raising np.linalg.LinAlgError (gram_schmidt.py:186-189)."""

import numpy as np
import pytest
import torch

import paper_2011_05090_b200 as sg

pytestmark = pytest.mark.gpu


def test_sketched_lsq_matches_lstsq(cuda, rng):
    # test_gram_schmidt.py:96-107, the HOUSEHOLDER_QR row (atol 1e-12)
    S = np.linalg.qr(rng.standard_normal((60, 8)))[0]
    S += 1e-4 * rng.standard_normal((60, 8))
    p = rng.standard_normal(60)
    oracle = np.linalg.lstsq(S, p, rcond=None)[0]
    y = sg.sketched_lsq(S, p, sg.HOUSEHOLDER_QR)
    assert isinstance(y, np.ndarray) and y.dtype == np.float64
    assert np.allclose(y, oracle, atol=1e-12)


@pytest.mark.parametrize("k,i", [(600, 300), (1500, 500), (2000, 37)])
def test_sketched_lsq_larger_bases(cuda, rng, k, i):
    """BASELINE-sized sketched bases (c0: 600 x 300, c1: 1500 x 500) with
    columns of mixed scale: the solution matches lstsq to 1e-10 relative."""
    S = np.linalg.qr(rng.standard_normal((k, i)))[0] * rng.uniform(0.5, 2.0, i)
    S += 1e-3 * rng.standard_normal((k, i))
    p = rng.standard_normal(k)
    oracle = np.linalg.lstsq(S, p, rcond=None)[0]
    y = sg.sketched_lsq(S, p)
    assert np.linalg.norm(y - oracle) <= 1e-10 * np.linalg.norm(oracle)


def test_sketched_lsq_fp32_and_device_io(cuda, rng):
    S = (np.linalg.qr(rng.standard_normal((200, 20)))[0]
         + 1e-3 * rng.standard_normal((200, 20))).astype(np.float32)
    p = rng.standard_normal(200)
    oracle = np.linalg.lstsq(S.astype(np.float64), p, rcond=None)[0]
    y = sg.sketched_lsq(S, p)
    assert y.dtype == np.float32
    assert np.linalg.norm(y - oracle) <= 1e-5 * np.linalg.norm(oracle)
    yd = sg.sketched_lsq(torch.from_numpy(S).cuda(), torch.from_numpy(p).cuda())
    assert isinstance(yd, torch.Tensor) and yd.is_cuda
    assert np.array_equal(yd.cpu().numpy(), y)


def test_sketched_lsq_rank_deficient(cuda, rng):
    # test_gram_schmidt.py:110-114: two identical columns and a zero column
    S = np.zeros((20, 3))
    S[:, 0] = S[:, 1] = rng.standard_normal(20)
    with pytest.raises(np.linalg.LinAlgError):
        sg.sketched_lsq(S, rng.standard_normal(20), sg.HOUSEHOLDER_QR)
    # a column in the span of the others (up to 1e-12): still rank deficient
    T = rng.standard_normal((50, 4))
    T[:, 3] = T[:, 0] - 2.0 * T[:, 2] + 1e-12 * rng.standard_normal(50)
    with pytest.raises(np.linalg.LinAlgError):
        sg.sketched_lsq(T, rng.standard_normal(50))


def test_sketched_lsq_edge_shapes(cuda, rng):
    assert sg.sketched_lsq(np.zeros((10, 0)), np.ones(10)).shape == (0,)
    with pytest.raises(ValueError):
        sg.sketched_lsq(rng.standard_normal((5, 5)), np.ones(5))  # i >= k
    with pytest.raises(ValueError):
        sg.sketched_lsq(rng.standard_normal((8, 2)), np.ones(7))
    with pytest.raises(NotImplementedError):
        sg.sketched_lsq(rng.standard_normal((8, 2)), np.ones(8), sg.LsqSolver("richardson"))


def test_pinned_result_buffers_are_owned(cuda):
    """rgs_factorize's pinned result buffers are reused only after the caller
    released every array/view of the previous result (weak ownership, no
    reference counting heuristics)."""
    import gc
    from paper_2011_05090_b200.workloads import make_w
    n, m, k = 8192, 8, 64
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 0)
    pin = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
    pin.copy_(torch.from_numpy(np.ascontiguousarray(make_w(n, m, 1e-2, 0).T)))
    W = pin.numpy().T
    pin2 = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
    pin2.copy_(2.0 * pin)
    W2 = pin2.numpy().T  # pinned and column-major: the pipelined path with pooled outputs
    f1, _ = sg.rgs_factorize(W, th, sg.UNIFIED64)
    Qview = f1.Q[:, 2:5]  # a view keeps the whole buffer owned
    keep = Qview.copy()
    del f1
    gc.collect()
    f2, _ = sg.rgs_factorize(W2, th, sg.UNIFIED64)
    assert np.array_equal(Qview, keep)        # not overwritten by the second call
    assert not np.shares_memory(Qview, f2.Q)
    from paper_2011_05090_b200 import gram_schmidt as gsm
    npool = len(gsm._PINNED_POOL)
    del f2, Qview
    gc.collect()
    f3, _ = sg.rgs_factorize(W, th, sg.UNIFIED64)
    assert len(gsm._PINNED_POOL) == npool  # released buffers reused, nothing newly pinned
    assert np.array_equal(f3.Q[:, 2:5], keep)
