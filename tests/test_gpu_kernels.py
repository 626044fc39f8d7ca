"""GPU numerics of the hand-written kernels through the C-ABI.

GEMM (tcgen05/TMEM/TMA): compared with an fp32 numpy product of the same
bf16 inputs. Tolerance: |dev - ref| <= 1e-2 * |ref| + 1e-2 * rms(ref)
(fp32 accumulation, bf16 output rounding = 2^-8 relative).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2507_06608_b200 import device
    return device


def _rand(D, rng, shape, scale=1.0):
    return D.f32_to_bf16(rng.standard_normal(shape).astype(np.float32) * scale)


def _close(dev, ref, rel=1e-2):
    tol = rel * np.abs(ref) + rel * np.sqrt(np.mean(ref * ref)) + 1e-6
    bad = np.abs(dev - ref) > tol
    assert not bad.any(), f"{bad.sum()} / {bad.size} out of tolerance; max err {np.abs(dev - ref).max()}"


SHAPES = [(1, 256, 256), (7, 768, 256), (33, 1024, 512), (64, 6144, 4096), (100, 2048, 1024),
          (300, 1024, 1024), (2048, 4096, 4096), (2100, 768, 256)]


@pytest.mark.parametrize("T,N,K", SHAPES)
def test_gemm_store(D, T, N, K):
    rng = np.random.default_rng(T * 7 + N)
    x, w = _rand(D, rng, (T, K)), _rand(D, rng, (N, K), 1 / np.sqrt(K))
    ref = D.bf16_to_f32(x) @ D.bf16_to_f32(w).T
    bx, bw, bo = D.Buf.from_array(x), D.Buf.from_array(w), D.Buf(T * N * 2)
    D.gemm(bx, bw, T, N, K, D.EPI_STORE, bo, N)
    _close(D.bf16_to_f32(bo.to_array((T, N), np.uint16)), ref)


@pytest.mark.parametrize("T,N,K,splits,sms", [(64, 1024, 4096, 4, 0), (5, 768, 2048, 3, 0),
                                              (200, 1024, 1024, 1, 3), (64, 4096, 4096, 0, 16)])
def test_gemm_splits_and_small_grids(D, T, N, K, splits, sms):
    rng = np.random.default_rng(5)
    x, w = _rand(D, rng, (T, K)), _rand(D, rng, (N, K), 1 / np.sqrt(K))
    ref = D.bf16_to_f32(x) @ D.bf16_to_f32(w).T
    bx, bw, bo = D.Buf.from_array(x), D.Buf.from_array(w), D.Buf(T * N * 2)
    D.gemm(bx, bw, T, N, K, D.EPI_STORE, bo, N, sm_count=sms, splits=splits)
    _close(D.bf16_to_f32(bo.to_array((T, N), np.uint16)), ref)


@pytest.mark.parametrize("T,N,K,sms", [(1024, 4096, 1024, 112), (2048, 6144, 512, 148), (700, 4096, 512, 40)])
def test_gemm_prefill_partial_waves(D, T, N, K, sms):
    """Prefill shapes whose last wave is partial on the partition: the runtime
    token-tile width (N in [192, 256]) refits the tiles to the waves
    (residual epilogue; the hybrid stream-K path runs with NX_HYBRID_FRAC)."""
    rng = np.random.default_rng(T + sms)
    x, w = _rand(D, rng, (T, K)), _rand(D, rng, (N, K), 1 / np.sqrt(K))
    r = _rand(D, rng, (T, N))
    ref = D.bf16_to_f32(x) @ D.bf16_to_f32(w).T + D.bf16_to_f32(r)
    bx, bw, br, bo = D.Buf.from_array(x), D.Buf.from_array(w), D.Buf.from_array(r), D.Buf(T * N * 2)
    D.gemm(bx, bw, T, N, K, D.EPI_RESIDUAL, bo, N, residual=br, ldr=N, sm_count=sms)
    _close(D.bf16_to_f32(bo.to_array((T, N), np.uint16)), ref)


@pytest.mark.parametrize("T,splits", [(9, 1), (64, 4), (500, 1)])
def test_gemm_bias_residual(D, T, splits):
    N, K = 1024, 1024
    rng = np.random.default_rng(T)
    x, w = _rand(D, rng, (T, K)), _rand(D, rng, (N, K), 1 / np.sqrt(K))
    b, r = _rand(D, rng, (N,)), _rand(D, rng, (T, N))
    bx, bw, bb, br = D.Buf.from_array(x), D.Buf.from_array(w), D.Buf.from_array(b), D.Buf.from_array(r)
    base = D.bf16_to_f32(x) @ D.bf16_to_f32(w).T
    for mode, ref in [(D.EPI_BIAS, base + D.bf16_to_f32(b)),
                      (D.EPI_RESIDUAL, base + D.bf16_to_f32(r)),
                      (D.EPI_BIAS_RESIDUAL, base + D.bf16_to_f32(b) + D.bf16_to_f32(r))]:
        bo = D.Buf(T * N * 2)
        D.gemm(bx, bw, T, N, K, mode, bo, N, bias=bb, residual=br, ldr=N, splits=splits)
        _close(D.bf16_to_f32(bo.to_array((T, N), np.uint16)), ref)


@pytest.mark.parametrize("T,splits", [(3, 1), (64, 4), (700, 1)])
def test_gemm_swiglu(D, T, splits):
    F, K = 1024, 512
    rng = np.random.default_rng(T + 1)
    x, w = _rand(D, rng, (T, K)), _rand(D, rng, (2 * F, K), 1 / np.sqrt(K))
    wf = D.bf16_to_f32(w).reshape(F // 64, 2, 64, K)
    g = D.bf16_to_f32(x) @ wf[:, 0].reshape(F, K).T
    u = D.bf16_to_f32(x) @ wf[:, 1].reshape(F, K).T
    ref = g / (1 + np.exp(-g)) * u
    bx, bw, bo = D.Buf.from_array(x), D.Buf.from_array(w), D.Buf(T * F * 2)
    D.gemm(bx, bw, T, 2 * F, K, D.EPI_SWIGLU, bo, F, splits=splits)
    _close(D.bf16_to_f32(bo.to_array((T, F), np.uint16)), ref)


@pytest.mark.parametrize("T,N,K,sms", [(1, 1024, 512, 0), (37, 4096 + 128, 4096, 0), (64, 4096, 4096, 48),
                                       (128, 6144, 4096, 16), (64, 4096, 14336, 148), (100, 28672, 4096, 0)])
def test_gemm_decode(D, T, N, K, sms):
    """Decode GEMM (tokens = MMA M, 256 weight rows = N): stream-K fold planes
    summed by the fold kernel, and the direct fp32 (data-parallel) form."""
    rng = np.random.default_rng(T + N)
    x, w = _rand(D, rng, (T, K)), _rand(D, rng, (N, K), 1 / np.sqrt(K))
    ref = D.bf16_to_f32(x) @ D.bf16_to_f32(w).T
    bx, bw = D.Buf.from_array(x), D.Buf.from_array(w)
    for mode in (D.EPI_DECODE_FOLD, D.EPI_DECODE_F32):
        bo = D.Buf(T * N * 4)
        D.gemm(bx, bw, T, N, K, mode, bo, N, sm_count=sms)
        dev = bo.to_array((T, N), np.float32)
        np.testing.assert_allclose(dev, ref, rtol=1e-3, atol=1e-3 * np.abs(ref).max())


@pytest.mark.parametrize("T,N,K,sms", [(300, 1024, 512, 148), (2048, 4096 + 128, 1024, 116), (700, 2048, 4096, 16)])
def test_gemm_pair_cta_group2(D, T, N, K, sms):
    """Prefill GEMM on CTA pairs (tcgen05 cta_group::2): store, residual and
    SwiGLU epilogues against the fp32 product."""
    rng = np.random.default_rng(T + N + K)
    x, w = _rand(D, rng, (T, K)), _rand(D, rng, (N, K), 1 / np.sqrt(K))
    r = _rand(D, rng, (T, N))
    base = D.bf16_to_f32(x) @ D.bf16_to_f32(w).T
    bx, bw, br = D.Buf.from_array(x), D.Buf.from_array(w), D.Buf.from_array(r)
    bo = D.Buf(T * N * 2)
    D.gemm(bx, bw, T, N, K, D.EPI_STORE, bo, N, sm_count=sms, splits=-2)
    _close(D.bf16_to_f32(bo.to_array((T, N), np.uint16)), base)
    D.gemm(bx, bw, T, N, K, D.EPI_RESIDUAL, bo, N, residual=br, ldr=N, sm_count=sms, splits=-2)
    _close(D.bf16_to_f32(bo.to_array((T, N), np.uint16)), base + D.bf16_to_f32(r))
    if N % 128 == 0:
        F = N // 2
        wf = D.bf16_to_f32(w).reshape(F // 64, 2, 64, K)
        g = D.bf16_to_f32(x) @ wf[:, 0].reshape(F, K).T
        u = D.bf16_to_f32(x) @ wf[:, 1].reshape(F, K).T
        bs = D.Buf(T * F * 2)
        D.gemm(bx, bw, T, N, K, D.EPI_SWIGLU, bs, F, sm_count=sms, splits=-2)
        _close(D.bf16_to_f32(bs.to_array((T, F), np.uint16)), g / (1 + np.exp(-g)) * u)


def test_gemm_f32_logits(D):
    T, N, K = 40, 1024 * 8, 512
    rng = np.random.default_rng(9)
    x, w = _rand(D, rng, (T, K)), _rand(D, rng, (N, K), 1 / np.sqrt(K))
    ref = D.bf16_to_f32(x) @ D.bf16_to_f32(w).T
    bx, bw, bo = D.Buf.from_array(x), D.Buf.from_array(w), D.Buf(T * N * 4)
    D.gemm(bx, bw, T, N, K, D.EPI_F32, bo, N)
    dev = bo.to_array((T, N), np.float32)
    np.testing.assert_allclose(dev, ref, rtol=1e-3, atol=1e-3 * np.abs(ref).max())


@pytest.mark.parametrize("T,N,K,sms,mode", [(64, 28672, 4096, 70, "swiglu"), (64, 4096, 14336, 37, "residual"),
                                            (17, 6144, 4096, 100, "bias"), (128, 1024, 512, 148, "f32"),
                                            (1, 128256 // 8 * 8, 512, 148, "f32")])
def test_gemm_streamk_partitions(D, T, N, K, sms, mode):
    """Decode-shaped launches on partial SM counts take the stream-K path
    (equal (tile, k-block) ranges per CTA + fix-up of split tiles)."""
    rng = np.random.default_rng(T + sms)
    x, w = _rand(D, rng, (T, K)), _rand(D, rng, (N, K), 1 / np.sqrt(K))
    b, r = _rand(D, rng, (N,)), _rand(D, rng, (T, N))
    xf, wf = D.bf16_to_f32(x), D.bf16_to_f32(w)
    bx, bw, bb, br = D.Buf.from_array(x), D.Buf.from_array(w), D.Buf.from_array(b), D.Buf.from_array(r)
    if mode == "swiglu":
        F = N // 2
        w4 = wf.reshape(F // 64, 2, 64, K)
        g, u = xf @ w4[:, 0].reshape(F, K).T, xf @ w4[:, 1].reshape(F, K).T
        ref = g / (1 + np.exp(-g)) * u
        bo = D.Buf(T * F * 2)
        D.gemm(bx, bw, T, N, K, D.EPI_SWIGLU, bo, F, sm_count=sms)
        _close(D.bf16_to_f32(bo.to_array((T, F), np.uint16)), ref)
        return
    base = xf @ wf.T
    if mode == "f32":
        bo = D.Buf(T * N * 4)
        D.gemm(bx, bw, T, N, K, D.EPI_F32, bo, N, sm_count=sms)
        np.testing.assert_allclose(bo.to_array((T, N), np.float32), base, rtol=1e-3,
                                   atol=1e-3 * np.abs(base).max())
        return
    m = {"residual": D.EPI_RESIDUAL, "bias": D.EPI_BIAS}[mode]
    ref = base + (D.bf16_to_f32(r) if mode == "residual" else D.bf16_to_f32(b))
    bo = D.Buf(T * N * 2)
    D.gemm(bx, bw, T, N, K, m, bo, N, bias=bb, residual=br, ldr=N, sm_count=sms)
    _close(D.bf16_to_f32(bo.to_array((T, N), np.uint16)), ref)
