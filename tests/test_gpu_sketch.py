"""GPU sketch kernels vs the reference golden vectors and the oracle."""

import math

import numpy as np
import pytest
import torch

import paper_2011_05090_b200 as sg
from conftest import golden
from oracle import OracleSketch

pytestmark = pytest.mark.gpu


def _relnorm(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def test_fwht_known_answer_and_dense(cuda):
    g = golden("fwht.npz")
    assert np.array_equal(sg.fwht(np.array([1.0, 2.0, 3.0, 4.0])), np.array([10.0, -2.0, -4.0, 0.0]))
    assert np.array_equal(sg.fwht(np.array([5.0])), np.array([5.0]))
    for s in (1, 2, 8, 64, 1024, 4096, 16384):
        y = sg.fwht(g[f"x_{s}"])
        # reference test_sketch.py:64-71 tolerance, and norm-wise ~log2(s) u
        assert np.max(np.abs(y - g[f"y_{s}"])) <= 1e-12 * s
        assert _relnorm(y, g[f"y_{s}"]) <= 1e-15 * max(1, math.log2(s))
    cols = np.stack([sg.fwht(g["X_mat"][:, j]) for j in range(3)], axis=1)
    assert np.array_equal(sg.fwht(g["X_mat"]), cols)  # axis-0, columnwise


def test_fwht_involution(cuda, rng):
    x = rng.standard_normal(256)
    assert np.allclose(sg.fwht(sg.fwht(x)) / 256.0, x, atol=1e-12)
    with pytest.raises(ValueError):
        sg.fwht(np.zeros(6))


def test_psrht_apply_matches_reference_golden(cuda):
    g = golden("psrht.npz")
    for (k, n, seed) in g["cases"]:
        tag = f"{k}_{n}_{seed}"
        op = sg.make_sketch(sg.SketchKind.PSRHT, int(k), int(n), int(seed))
        y = op.apply(g[f"x_{tag}"])
        assert y.dtype == np.float64 and y.shape == (int(k),)
        # norm-wise relative 1e-14: GPU and numpy butterfly orders differ (~log2 s * u)
        assert _relnorm(y, g[f"y_{tag}"]) <= 1e-14, tag
        Y = op.apply_block(g[f"X_{tag}"])
        assert _relnorm(Y, g[f"Y_{tag}"]) <= 1e-14, tag


def test_apply_block_bit_identical_to_apply(cuda, rng):
    for kind, k, n in ((sg.SketchKind.PSRHT, 20, 50), (sg.SketchKind.PSRHT, 300, 70000),
                       (sg.SketchKind.RADEMACHER, 20, 50), (sg.SketchKind.GAUSSIAN, 64, 9000)):
        th = sg.make_sketch(kind, k, n, seed=5)
        X = rng.standard_normal((n, 4))
        blk = th.apply_block(X)
        for j in range(4):
            assert np.array_equal(blk[:, j], th.apply(X[:, j])), kind


def test_determinism_and_seed_dependence(cuda):
    x = np.random.default_rng(3).standard_normal(100)
    for kind in (sg.SketchKind.PSRHT, sg.SketchKind.RADEMACHER, sg.SketchKind.GAUSSIAN):
        a = sg.make_sketch(kind, 40, 100, seed=11).apply(x)
        b = sg.make_sketch(kind, 40, 100, seed=11).apply(x)
        c = sg.make_sketch(kind, 40, 100, seed=12).apply(x)
        assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_entries_and_materialize(cuda):
    g = golden("psrht.npz")
    th = sg.make_sketch(sg.SketchKind.PSRHT, 16, 24, seed=0)
    M = th.materialize()
    assert M.shape == (16, 24)
    assert np.allclose(np.abs(M), 1.0 / 4.0)
    assert np.allclose(M, g["materialize_16_24_0"], atol=1e-15)
    R = sg.make_sketch(sg.SketchKind.RADEMACHER, 20, 50, 5).materialize()
    assert np.allclose(R, g["rad_materialize_20_50_5"], atol=1e-15)


def test_shape_validation(cuda):
    th = sg.make_sketch(sg.SketchKind.PSRHT, 4, 10, seed=0)
    with pytest.raises(ValueError):
        th.apply(np.zeros(11))
    with pytest.raises(ValueError):
        th.apply_block(np.zeros((11, 2)))


def test_dense_and_block_kinds_vs_oracle(cuda, rng):
    for kind, k, n, kw in (("gaussian", 600, 20000, {}), ("rademacher", 64, 3000, {}),
                           ("block_srht", 200, 8 * 2048, {"block_log2": 11})):
        op = sg.make_sketch(sg.SketchKind(kind), k, n, 7, **kw)
        orc = OracleSketch(kind, k, n, 7, **kw)
        x = rng.standard_normal(n)
        assert _relnorm(op.apply(x), orc.apply(x)) <= 1e-14, kind


def test_device_tensor_io_and_fp32_input(cuda, rng):
    th = sg.make_sketch(sg.SketchKind.PSRHT, 150, 100_000, 1)
    x = rng.standard_normal(100_000).astype(np.float32)
    y_host = th.apply(x)  # numpy path (coerced to fp64 like sketch.py:170)
    y_dev = th.apply(torch.from_numpy(x).cuda())  # fp32 read in-kernel, exact upcast
    assert isinstance(y_dev, torch.Tensor) and y_dev.dtype == torch.float64
    assert np.array_equal(y_dev.cpu().numpy(), y_host)


def test_large_psrht_linearity_and_norm(cuda):
    # full c1 size: n = 1e6, s = 2^20, k = 1500; size-independent properties
    n, k = 1_000_000, 1500
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 1)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    z = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    yx, yz = th.apply(x), th.apply(z)
    yxz = th.apply(2.0 * x - 3.0 * z)
    lin = torch.linalg.norm(yxz - (2.0 * yx - 3.0 * yz)) / torch.linalg.norm(yxz)
    assert float(lin) < 1e-13
    # E||Theta x||^2 = ||x||^2 for the reference scaling 1/sqrt(k) of the unnormalised H
    ratio = float(torch.linalg.norm(yx) / torch.linalg.norm(x))
    assert 0.9 < ratio < 1.1
    # bit-identical rerun
    assert torch.equal(th.apply(x), yx)


@pytest.mark.parametrize("k,n,seed", [(64, 3000, 5), (601, 2000, 11), (1500, 700, 3)])
def test_device_rademacher_bits_match_reference_streams(cuda, k, n, seed):
    """sgs_rademacher_bits reproduces the reference's per-column streams
    Philox((seed << 64) | j).integers(0, 2, size=k) (sketch.py:153-158) bit for bit."""
    from oracle.ref_sketch import _gen
    th = sg.make_sketch(sg.SketchKind.RADEMACHER, k, n, seed)
    words = th.device_data()["rbits"].cpu().numpy().view(np.uint32)
    bits = np.unpackbits(words.view(np.uint8), axis=1, bitorder="little")[:, :k]
    ref = np.stack([_gen(seed, j).integers(0, 2, size=k) for j in range(n)])
    assert np.array_equal(bits, ref)
    # packed-sign partials == the dense fp64 definition, bit for bit on exact inputs
    rng = np.random.default_rng(1)
    X = rng.integers(-8, 8, size=(n, 3)).astype(np.float64)
    Y = th.apply_block(X)
    assert np.array_equal(Y, th.scale * ((2.0 * ref.T - 1.0) @ X))  # exact integer sums
    Xr = rng.standard_normal((n, 2))
    assert np.allclose(th.apply_block(Xr), (2.0 * ref.T - 1.0) @ Xr / np.sqrt(k), rtol=1e-13,
                       atol=1e-13)
    y0 = th.apply(Xr[:, 0])
    assert np.array_equal(y0, th.apply_block(Xr)[:, 0])  # apply_block == apply


@pytest.mark.parametrize("dt,n,kind", [(torch.float64, 1_000_000, "psrht"),
                                       (torch.float32, 3 * 4096 + 100, "psrht"),
                                       (torch.float64, 4 * 4096, "block_srht")])
def test_column_kernel_sketch_equals_stand_alone_sketch(cuda, dt, n, kind):
    """The fused column kernel's SRHT epilogue and the stand-alone tile kernel
    run the same transform (stage order bits 6..11 then 0..5, one tile per
    CTA, 8-CTA cluster sums): for column 0 (q'_0 = w) their partials are
    bit-identical, so the S of a factorisation equals Theta applied to the
    unnormalised basis exactly as apply() would compute it."""
    from paper_2011_05090_b200 import _lib
    kw = {"block_log2": 12} if kind == "block_srht" else {}
    th = sg.make_sketch(sg.SketchKind(kind), 300, n, 7, **kw)
    d = th.device_data(cuda)
    code = _lib.dtype_code(dt)
    w = torch.randn(n, dtype=torch.float64, device=cuda, generator=torch.Generator(cuda).manual_seed(1)).to(dt)
    ldq = (n + 31) // 32 * 32
    Q = torch.zeros((2, ldq), dtype=dt, device=cuda)
    npc = int(_lib.load().sgs_column_nparts(n))
    assert npc == th.nparts(n)
    pc = torch.empty((npc, th.k), dtype=torch.float64, device=cuda)
    ps = torch.empty_like(pc)
    st = _lib.Status(cuda)
    _lib.call("sgs_rgs_update_srht", Q.data_ptr(), code, ldq, n, 0, w.data_ptr(), code, None,
              None, 0, None, 2, 1, 0, th.log2_block, d["bits"].data_ptr(),
              d["samples"].data_ptr(), th.k, pc.data_ptr(), st.ptr, _lib.stream_ptr())
    th.partials_into(w, code, n, 1, ps, status=st)
    torch.cuda.synchronize()
    assert torch.equal(Q[0, :n], w)
    assert torch.equal(pc, ps)


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_batched_tile_sketch_equals_per_column(cuda, dt):
    """Batches of many columns run srht_tile3_kernel: one 256-thread CTA per
    tile group, tiles in order, three register phases of the same butterfly
    levels in the same order; single columns run the 64-thread tile kernel,
    one tile per CTA with a DSMEM cluster sum.  Same partial structure and
    order: apply_block over 24 columns of c1's shape equals 24 apply() calls
    bit for bit."""
    n, k, m = 1_000_000, 1500, 24
    th = sg.make_sketch(sg.SketchKind.PSRHT, k, n, 2)
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g).to(dt)
    Y = th.apply_block(X.t())
    for j in range(m):
        assert torch.equal(Y[:, j], th.apply(X[j]))


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_batched_block_srht_equals_per_column(cuda, dt):
    """Batch mode with a block-SRHT of 4096-row blocks: every tile of a CTA's
    eight switches sample rows (and the fp32 path prefetches the next tile's
    values and sign words while transforming the current one); a ragged last
    block-row is zero padded.  apply_block equals apply bit for bit."""
    n, k, m = 64 * 4096, 700, 80
    th = sg.make_sketch(sg.SketchKind.BLOCK_SRHT, k, n, 9, block_log2=12)
    g = torch.Generator(device="cuda").manual_seed(11)
    X = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g).to(dt)
    Y = th.apply_block(X.t())
    for j in range(0, m, 7):
        assert torch.equal(Y[:, j], th.apply(X[j]))


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_gaussian_dmma_batch_equals_per_column(cuda, dt):
    """The Gaussian P = Theta W on the fp64 tensor cores: the 128 x 64 tile
    variant (batches) and the 256 x 8 variant (apply) run the same ascending
    4-row DMMA chains per output - DMMA evaluates its four products as a
    sequential fma chain (tools/dmma_probe.py) - so apply_block equals apply
    bit for bit, and both match the oracle's fp64 GEMV to rounding."""
    n, k, m = 100_000, 600, 20
    th = sg.make_sketch(sg.SketchKind.GAUSSIAN, k, n, 3)
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g).to(dt)
    Y = th.apply_block(X.t())
    for j in range(m):
        assert torch.equal(Y[:, j], th.apply(X[j]))
    orc = OracleSketch("gaussian", k, n, 3)
    ref = orc.apply(X[0].double().cpu().numpy())
    assert _relnorm(Y[:, 0].cpu().numpy(), ref) <= 1e-14
