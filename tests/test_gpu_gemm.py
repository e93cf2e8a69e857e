"""tcgen05 GEMM kernel against a plain fp32 reference of the same op (bf16 operands
rounded identically on both sides), for every operand major-ness the DASH step
uses: (K,K) forward projections, (K,MN) input gradients, (MN,MN) weight gradients."""
import numpy as np
import pytest

import paper_2505_17218_b200 as D

pytestmark = pytest.mark.gpu


def bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


@pytest.fixture(scope="module")
def ctx():
    return D.Context(0)


SHAPES = [(128, 128, 64), (256, 384, 128), (200, 136, 72), (77, 300, 1000), (1024, 896, 896), (36, 1152, 896),
          (896, 4864, 517), (4096, 4864, 256), (2000, 1152, 300), (3000, 2048, 128)]   # last 3: several tiles/CTA


@pytest.mark.parametrize("ak", [True, False])
@pytest.mark.parametrize("bk", [True, False])
@pytest.mark.parametrize("shape", SHAPES)
def test_tc_gemm_matches_fp32_reference(ctx, ak, bk, shape):
    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = bf16_bits(rng.standard_normal((M, K)).astype(np.float32))
    B = bf16_bits(rng.standard_normal((N, K)).astype(np.float32))
    ref = bits_to_f32(A).astype(np.float64) @ bits_to_f32(B).astype(np.float64).T
    Ast = A if ak else np.ascontiguousarray(A.T)
    Bst = B if bk else np.ascontiguousarray(B.T)
    # strides must be 16-byte multiples for TMA; pad the leading dimension when needed
    def pad(x):
        cols = x.shape[1]
        p = (-cols) % 8
        return np.pad(x, ((0, 0), (0, p))) if p else x
    Ast, Bst = pad(Ast), pad(Bst)
    got = ctx.selftest_gemm(Ast, ak, Bst, bk, M, N, K)
    err = np.abs(got - ref).max() / max(1.0, np.abs(ref).max())
    assert err < 1e-5, err


def test_tc_gemm_epilogues(ctx):
    M, N, K = 192, 256, 320
    rng = np.random.default_rng(0)
    A = bf16_bits(rng.standard_normal((M, K)).astype(np.float32) * 0.1)
    B = bf16_bits(rng.standard_normal((N, K)).astype(np.float32) * 0.1)
    bias = rng.standard_normal(N).astype(np.float32)
    ref = bits_to_f32(A).astype(np.float64) @ bits_to_f32(B).astype(np.float64).T
    got = ctx.selftest_gemm(A, True, B, True, M, N, K, bias=bias, epi=1)
    assert np.abs(got - np.tanh(ref + bias)).max() < 1e-3   # tanh.approx: 2^-10.99 relative
    c0 = rng.standard_normal((M, N)).astype(np.float32)
    got = ctx.selftest_gemm(A, True, B, True, M, N, K, epi=3, C_init=c0)
    assert np.abs(got - (c0 + ref)).max() < 1e-4


def test_tc_matches_simt(ctx):
    M, N, K = 300, 500, 260
    rng = np.random.default_rng(1)
    A = bf16_bits(rng.standard_normal((M, K)).astype(np.float32))
    B = bf16_bits(rng.standard_normal((K, N)).astype(np.float32))
    a = ctx.selftest_gemm(A, True, B, False, M, N, K)
    b = ctx.selftest_gemm(A, True, B, False, M, N, K, force_simt=True)
    assert np.abs(a - b).max() <= 1e-4 * np.abs(b).max()


@pytest.mark.parametrize("shape", [(200, 136, 72), (77, 300, 1000), (3000, 2048, 128)])
@pytest.mark.parametrize("epi", [0, 1, 3, 4])
def test_tma_store_epilogue_matches_direct_stores(ctx, knob, shape, epi):
    """The bulk-tensor-store epilogue (and its fp32 reduce-add for EPI_ACCUM) writes
    exactly what the per-thread 16-byte stores write, ragged edges included."""
    M, N, K = shape
    rng = np.random.default_rng(5)
    A = bf16_bits(rng.standard_normal((M, K)).astype(np.float32) * 0.1)
    B = bf16_bits(rng.standard_normal((N, K)).astype(np.float32) * 0.1)
    bias = rng.standard_normal(N).astype(np.float32)
    c0 = rng.standard_normal((M, N)).astype(np.float32)
    kw = dict(bias=bias if epi != 3 else None, epi=epi, C_init=c0 if epi in (3, 4) else None)
    got = ctx.selftest_gemm(A, True, B, True, M, N, K, **kw)
    knob("NO_TMA_STORE", "1")
    ref = ctx.selftest_gemm(A, True, B, True, M, N, K, **kw)
    if epi == 1:  # the direct path's ragged columns use the scalar epilogue (precise tanhf);
        # the vector paths use MUFU tanh.approx (max relative error 2^-10.99, below bf16 rounding)
        assert np.abs(got - ref).max() < 1e-3
        full = (N // 32) * 32
        assert np.array_equal(got[:, :full].view(np.uint32), ref[:, :full].view(np.uint32))
    else:
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("pair", ["-1", "0", "3"])
@pytest.mark.parametrize("raster", ["0", "1"])
@pytest.mark.parametrize("shape", [(128, 128, 8192), (896, 896, 36832 // 8), (300, 200, 5000), (4864, 896, 4096)])
def test_split_k_accumulate(ctx, knob, shape, raster, pair):
    """Weight-gradient shapes (few output tiles, long K) run as ordered split-K (single-CTA
    and CTA-pair kernels): the slices reduce into C in slice order, so repeated runs are
    bit-identical and the result matches the unsplit kernel to fp32 rounding."""
    knob("GEMM_RASTER", raster)
    knob("GEMM_PAIR", pair)   # -1 single-CTA split-K, 3: 256x224 pair split-K
    M, N, K = shape
    rng = np.random.default_rng(11)
    A = bf16_bits(rng.standard_normal((K, M)).astype(np.float32))   # MN-major operands, as in dW = dY^T X
    B = bf16_bits(rng.standard_normal((K, N)).astype(np.float32))
    c0 = rng.standard_normal((M, N)).astype(np.float32)
    ref = c0 + bits_to_f32(A).astype(np.float64).T @ bits_to_f32(B).astype(np.float64)
    a = ctx.selftest_gemm(A, False, B, False, M, N, K, epi=3, C_init=c0)
    b = ctx.selftest_gemm(A, False, B, False, M, N, K, epi=3, C_init=c0)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.abs(a - ref).max() <= 1e-5 * np.abs(ref).max() + 1e-3
    knob("NO_SPLITK", "1")
    c = ctx.selftest_gemm(A, False, B, False, M, N, K, epi=3, C_init=c0)
    assert np.abs(a - c).max() <= 1e-5 * np.abs(ref).max() + 1e-3


@pytest.mark.parametrize("raster", ["0", "1"])
@pytest.mark.parametrize("pair", ["1", "2", "3", "-1"])
@pytest.mark.parametrize("ak,bk", [(True, True), (True, False), (False, True), (False, False)])
@pytest.mark.parametrize("shape", [(256, 128, 64), (300, 200, 136), (4096, 896, 896), (1000, 1152, 320),
                                   (520, 448, 200)])
def test_cta_pair_tiles(ctx, knob, pair, ak, bk, shape, raster):
    """The cta_group::2 kernel with 256x256 (pair=1), 256x128 (pair=2) and 256x224 (pair=3)
    tiles, forced, and the single-CTA kernel (pair=-1), under both tile rasters."""
    knob("GEMM_PAIR", pair)
    knob("GEMM_RASTER", raster)
    M, N, K = shape
    rng = np.random.default_rng(M + N + K)
    A = bf16_bits(rng.standard_normal((M, K)).astype(np.float32))
    B = bf16_bits(rng.standard_normal((N, K)).astype(np.float32))
    ref = bits_to_f32(A).astype(np.float64) @ bits_to_f32(B).astype(np.float64).T
    Ast = A if ak else np.ascontiguousarray(A.T)
    Bst = B if bk else np.ascontiguousarray(B.T)
    got = ctx.selftest_gemm(Ast, ak, Bst, bk, M, N, K)
    assert np.abs(got - ref).max() / max(1.0, np.abs(ref).max()) < 1e-5


@pytest.mark.parametrize("pair", ["1", "3"])
@pytest.mark.parametrize("deep", ["0", "1"])
@pytest.mark.parametrize("shape", [(300, 200, 136), (4096, 896, 896), (1000, 1152, 320)])
def test_pair_residual_prefetch_epilogue(ctx, knob, shape, deep, pair):
    """The CTA-pair kernel's double-buffered residual epilogue (fp32 resid in, fp32 out)
    equals the per-thread direct-store epilogue bit-for-bit, ragged edges included."""
    M, N, K = shape
    rng = np.random.default_rng(17)
    A = bf16_bits(rng.standard_normal((M, K)).astype(np.float32) * 0.1)
    B = bf16_bits(rng.standard_normal((N, K)).astype(np.float32) * 0.1)
    bias = rng.standard_normal(N).astype(np.float32)
    c0 = rng.standard_normal((M, N)).astype(np.float32)
    knob("GEMM_PAIR", pair)
    knob("GEMM_RESID_DEEP", deep)   # 5 stages x 4 epilogue warps
    got = ctx.selftest_gemm(A, True, B, True, M, N, K, bias=bias, epi=4, C_init=c0)
    knob("GEMM_RESID_DB", "0")
    mid = ctx.selftest_gemm(A, True, B, True, M, N, K, bias=bias, epi=4, C_init=c0)
    knob("NO_TMA_STORE", "1")
    ref = ctx.selftest_gemm(A, True, B, True, M, N, K, bias=bias, epi=4, C_init=c0)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    assert np.array_equal(mid.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("M", [1, 8, 32, 33, 64, 100])
@pytest.mark.parametrize("NK", [(896, 4864), (1152, 896), (4864, 896)])
def test_skinny_rows_equal_big_batch_rows(ctx, knob, M, NK):
    """A decode step at a few rows (the skinny path: 32- / 64-row A boxes, deep rings)
    computes every row bit-identically to the same row inside a 4096-row batch (other
    tile shapes, CTA pairs) and to the full 128-row-box path: a sequence's tokens do not
    depend on how many sequences share its decode batch."""
    N, K = NK
    rng = np.random.default_rng(M + N + K)
    A = bf16_bits(rng.standard_normal((4096, K)).astype(np.float32) * 0.1)
    B = bf16_bits(rng.standard_normal((N, K)).astype(np.float32) * 0.1)
    bias = rng.standard_normal(N).astype(np.float32)
    c0 = rng.standard_normal((4096, N)).astype(np.float32)
    for epi in (1, 4):   # tanh (W1) and the residual-stream store (Wo / W2)
        kw = dict(bias=bias, epi=epi)
        big = ctx.selftest_gemm(A, True, B, True, 4096, N, K, C_init=c0 if epi == 4 else None, **kw)
        small = ctx.selftest_gemm(A[:M], True, B, True, M, N, K, C_init=c0[:M] if epi == 4 else None, **kw)
        assert np.array_equal(small.view(np.uint32), big[:M].view(np.uint32)), epi
        knob("GEMM_SKINNY_AR", "0")
        full = ctx.selftest_gemm(A[:M], True, B, True, M, N, K, C_init=c0[:M] if epi == 4 else None, **kw)
        knob("GEMM_SKINNY_AR", None)
        assert np.array_equal(small.view(np.uint32), full.view(np.uint32)), epi


@pytest.mark.parametrize("M", [1, 16, 32, 33, 64])
@pytest.mark.parametrize("NK", [(896, 4864), (1152, 896), (4864, 896)])
def test_skinny_m64_mma_rows_equal_big_batch_rows(ctx, knob, M, NK):
    """The M = 64 MMA form of the skinny path (KNOB_GEMM_SKINNY_M64: accumulator rows in
    TMEM lanes 0-15 of each quarter) gives the same bits as the same rows in a 4096-row batch."""
    N, K = NK
    rng = np.random.default_rng(M * 3 + N + K)
    A = bf16_bits(rng.standard_normal((4096, K)).astype(np.float32) * 0.1)
    B = bf16_bits(rng.standard_normal((N, K)).astype(np.float32) * 0.1)
    bias = rng.standard_normal(N).astype(np.float32)
    c0 = rng.standard_normal((4096, N)).astype(np.float32)
    for epi in (1, 4):
        kw = dict(bias=bias, epi=epi)
        big = ctx.selftest_gemm(A, True, B, True, 4096, N, K, C_init=c0 if epi == 4 else None, **kw)
        knob("GEMM_SKINNY_M64", "1")
        small = ctx.selftest_gemm(A[:M], True, B, True, M, N, K, C_init=c0[:M] if epi == 4 else None, **kw)
        knob("GEMM_SKINNY_M64", None)
        assert np.array_equal(small.view(np.uint32), big[:M].view(np.uint32)), (epi, np.abs(small - big[:M]).max())


@pytest.mark.parametrize("pair", ["0", "-1", "1", "2", "3"])
@pytest.mark.parametrize("shape", [(1, 8, 16), (33, 72, 40), (65, 904, 200), (129, 264, 64), (257, 1160, 72),
                                   (300, 4872, 64), (511, 896, 1096)])
@pytest.mark.parametrize("epi", [0, 1, 3, 4])
def test_ragged_tiles_stay_inside_the_output(ctx, knob, pair, shape, epi):
    """Every kernel family (skinny M = 64 / 128-row, single-CTA 128 / 256 wide, CTA pairs
    256 / 128 / 224 wide, split-K accumulate) on ragged M / N / K: selftest_gemm surrounds C
    with 0xA5 guard bands (16 KB before, 256 rows after) and fails if any epilogue store
    lands outside C (our stand-in for compute-sanitizer memcheck, closed on the GPU pool);
    the values match the fp64 reference."""
    knob("GEMM_PAIR", pair)
    M, N, K = shape
    rng = np.random.default_rng(M * 31 + N + K + epi)
    A = bf16_bits(rng.standard_normal((M, K)).astype(np.float32) * 0.1)
    B = bf16_bits(rng.standard_normal((N, K)).astype(np.float32) * 0.1)
    bias = rng.standard_normal(N).astype(np.float32)
    c0 = rng.standard_normal((M, N)).astype(np.float32)
    ref = bits_to_f32(A).astype(np.float64) @ bits_to_f32(B).astype(np.float64).T
    if epi == 3:   # accumulate (weight-gradient form, MN-major operands)
        def pad(x):   # 16-byte row pitch for the TMA maps (the padding columns lie outside M / N)
            p = (-x.shape[1]) % 8
            return np.pad(x, ((0, 0), (0, p))) if p else x
        got = ctx.selftest_gemm(pad(np.ascontiguousarray(A.T)), False, pad(np.ascontiguousarray(B.T)), False, M, N, K,
                                epi=3, C_init=c0)
        want, tol = c0 + ref, 1e-4
    else:
        got = ctx.selftest_gemm(A, True, B, True, M, N, K, bias=bias if epi else None, epi=epi,
                                C_init=c0 if epi == 4 else None)
        want = {0: ref, 1: np.tanh(ref + bias), 4: c0 + ref + bias}[epi]
        tol = 1e-3 if epi == 1 else 1e-4
    assert np.abs(got - want).max() < tol
