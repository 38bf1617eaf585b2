"""Per-kernel parity: the tcgen05 implicit-GEMM conv against the CPU oracle.

Operands are TF32-rounded before both paths see them, so the only difference
left is fp32 accumulation order inside the tensor core: tolerance 2e-5
relative to max|ref| (written here, per the north_star's fp32 tolerance
budget of 1e-3 end to end).
"""
import numpy as np
import pytest

from oracle.layers import conv2d_nhwc, round_tf32

TOL = 2e-5


def run_conv(nimg, H, W, Cin, N, KH, KW, stride, pad, *, in_ldc=None, in_coff=0, out_ldc=None,
             out_coff=0, residual=False, relu=0, bias=True, seed=0, round_out=0, split=0, raw_input=False,
             bf16_ref=False):
    """Runs the conv kernel through the C-ABI test hook; returns max|gpu - ref|
    / max|ref|. split: 0 TF32, 1 2xTF32, 2 BF16. bf16_ref: the reference sees
    the operands rounded to bf16 (what the BF16 path multiplies), so only the
    fp32 accumulation order differs."""
    from paper_2304_09961_b200._native import bs_conv_desc, check, exec_lib, fptr
    rng = np.random.default_rng(seed)
    in_ldc = in_ldc or Cin
    out_ldc = out_ldc or N
    Ho = (H + 2 * pad - KH) // stride + 1
    Wo = (W + 2 * pad - KW) // stride + 1
    x_full = rng.standard_normal((nimg, H, W, in_ldc)).astype(np.float32)
    if not raw_input:
        x_full = round_tf32(x_full)
    x = x_full[..., in_coff:in_coff + Cin]
    w = round_tf32((rng.standard_normal((N, KH, KW, Cin)) / np.sqrt(KH * KW * Cin)).astype(np.float32))
    K = KH * KW * Cin
    Kpad = (K + 31) // 32 * 32
    wp = np.zeros((N, Kpad), np.float32)
    wp[:, :K] = w.reshape(N, K)
    b = rng.standard_normal(N).astype(np.float32) if bias else None
    res_full = rng.standard_normal((nimg, Ho, Wo, out_ldc)).astype(np.float32) if residual else None
    out = np.full((nimg, Ho, Wo, out_ldc), 7.0, np.float32)

    if bf16_ref:
        from oracle.layers import round_bf16
        ref = conv2d_nhwc(round_bf16(x), round_bf16(w), b, stride, pad)
    else:
        ref = conv2d_nhwc(x, w, b, stride, pad)
    if residual:
        ref = ref + res_full[..., out_coff:out_coff + N]
    if relu == 1:
        ref = np.maximum(ref, 0)
    elif relu == 2:
        ref = np.clip(ref, 0, 6)

    d = bs_conv_desc(H=H, W=W, Cin=Cin, Ho=Ho, Wo=Wo, KH=KH, KW=KW, stride=stride, pad=pad, N=N,
                     in_ldc=in_ldc, in_coff=in_coff, out_ldc=out_ldc, out_coff=out_coff,
                     res_ldc=out_ldc, res_coff=out_coff, relu=relu, round_out=round_out, split=split)
    lib = exec_lib()
    check(lib.bs_kernel_conv(d, nimg, fptr(x_full), fptr(wp), fptr(b), fptr(res_full), fptr(out), 0,
                             None))
    got = out[..., out_coff:out_coff + N]
    err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)
    # untouched channels keep the sentinel
    if out_ldc > N:
        mask = np.ones(out_ldc, bool)
        mask[out_coff:out_coff + N] = False
        assert np.all(out[..., mask] == 7.0)
    return err


CASES = [
    dict(nimg=2, H=14, W=14, Cin=64, N=128, KH=1, KW=1, stride=1, pad=0),
    dict(nimg=3, H=28, W=28, Cin=64, N=96, KH=3, KW=3, stride=1, pad=1),
    dict(nimg=1, H=15, W=15, Cin=32, N=64, KH=3, KW=3, stride=2, pad=1),
    dict(nimg=2, H=32, W=32, Cin=4, N=64, KH=7, KW=7, stride=2, pad=3),
    dict(nimg=5, H=1, W=1, Cin=1024, N=1000, KH=1, KW=1, stride=1, pad=0),
    dict(nimg=1, H=7, W=7, Cin=832, N=384, KH=1, KW=1, stride=1, pad=0),
    dict(nimg=4, H=7, W=7, Cin=160, N=320, KH=3, KW=3, stride=1, pad=1),
    dict(nimg=2, H=9, W=9, Cin=24, N=16, KH=1, KW=1, stride=1, pad=0),
    dict(nimg=3, H=1, W=1, Cin=128, N=10, KH=1, KW=1, stride=1, pad=0),
    dict(nimg=2, H=14, W=14, Cin=64, N=48, KH=1, KW=1, stride=2, pad=0),
    # small channel counts, odd batches, stride 2
    dict(nimg=3, H=7, W=7, Cin=16, N=32, KH=3, KW=3, stride=1, pad=1),
    dict(nimg=2, H=14, W=14, Cin=48, N=64, KH=3, KW=3, stride=1, pad=1),
    dict(nimg=2, H=56, W=56, Cin=24, N=144, KH=1, KW=1, stride=1, pad=0),
    dict(nimg=2, H=112, W=112, Cin=16, N=32, KH=3, KW=3, stride=2, pad=1),
    dict(nimg=5, H=8, W=8, Cin=64, N=64, KH=3, KW=3, stride=1, pad=1),
    # Tap-row mode (stems: one K tile per filter row): tiles inside one image
    # and across images (HoWo < 128 and not a multiple of 128), Cin 8 / 16.
    dict(nimg=3, H=100, W=100, Cin=4, N=64, KH=7, KW=7, stride=2, pad=3),
    dict(nimg=5, H=16, W=16, Cin=4, N=64, KH=7, KW=7, stride=2, pad=3),
    dict(nimg=3, H=30, W=30, Cin=8, N=48, KH=3, KW=3, stride=1, pad=1),
    dict(nimg=2, H=20, W=20, Cin=16, N=32, KH=1, KW=1, stride=1, pad=0),
    dict(nimg=2, H=9, W=11, Cin=16, N=40, KH=2, KW=2, stride=1, pad=0),
    # Row-window stems (Wo >= 64: a tile's <= 3 input rows bulk-copied per
    # filter row): tiles across images, Cin 4 / 8 / 16, batch 1 (split-K).
    dict(nimg=3, H=150, W=150, Cin=4, N=64, KH=7, KW=7, stride=2, pad=3),
    dict(nimg=1, H=224, W=224, Cin=4, N=64, KH=7, KW=7, stride=2, pad=3),
    dict(nimg=2, H=130, W=130, Cin=8, N=48, KH=3, KW=3, stride=1, pad=1),
    dict(nimg=2, H=66, W=70, Cin=16, N=32, KH=2, KW=2, stride=1, pad=0),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(str(c[k]) for k in ("nimg", "H", "Cin", "N", "KH", "stride")))
def test_conv_matches_oracle(case):
    assert run_conv(**case) < TOL


@pytest.mark.gpu
def test_conv_channel_slices_residual_relu():
    err = run_conv(2, 14, 14, 64, 96, 3, 3, 1, 1, in_ldc=256, in_coff=64, out_ldc=512,
                   out_coff=128, residual=True, relu=1)
    assert err < TOL


@pytest.mark.gpu
def test_conv_stem_tap_rows_residual_relu():
    # Full-width stem rows (224 -> 112, two images per some tiles) with a residual.
    assert run_conv(2, 224, 224, 4, 64, 7, 7, 2, 3, residual=True, relu=1) < TOL


@pytest.mark.gpu
def test_conv_relu6():
    assert run_conv(2, 8, 8, 32, 64, 1, 1, 1, 0, relu=2) < TOL


@pytest.mark.gpu
def test_conv_large_batch():
    assert run_conv(90, 7, 7, 256, 256, 3, 3, 1, 1, bias=False) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES[:7], ids=lambda c: "x".join(str(c[k]) for k in ("nimg", "H", "Cin", "N", "KH", "stride")))
def test_conv_split_tf32x2_full_fp32_inputs(case):
    """2xTF32: un-rounded fp32 activations, TF32 weights -> fp32-level error."""
    assert run_conv(**case, split=1, raw_input=True) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES[:10] + CASES[15:], ids=lambda c: "x".join(str(c[k]) for k in ("nimg", "H", "Cin", "N", "KH", "stride")))
def test_conv_bf16_operands(case):
    """BF16 precision (kind::f16 MMAs, A rounded to bf16 by the converters,
    bf16 weight copies by 64B-swizzled TMA): exact bf16 products with fp32
    accumulation -- 2e-5 against a reference on bf16-rounded operands, and
    within bf16 rounding (1e-2) of the fp32 result."""
    assert run_conv(**case, split=2, raw_input=True, bf16_ref=True) < TOL
    assert run_conv(**case, split=2, raw_input=True) < 1e-2


@pytest.mark.gpu
@pytest.mark.parametrize("split", [1, 2])
def test_conv_cluster_split_k_forced(split, monkeypatch):
    """Every K split the autotune may force (cluster of 2..8 CTAs per tile,
    DSMEM reduction), including ragged K tiles per split."""
    for ks in ("2", "3", "5", "8"):
        monkeypatch.setenv("BS_CONV_KS_FORCE", ks)
        assert run_conv(1, 7, 7, 832, 384, 1, 1, 1, 0, split=split, raw_input=True,
                        bf16_ref=split == 2, residual=True, relu=1) < TOL
        assert run_conv(3, 14, 14, 96, 208, 3, 3, 1, 1, split=split, raw_input=True, bf16_ref=split == 2) < TOL


@pytest.mark.gpu
def test_conv_plain_tf32_on_fp32_inputs_is_worse():
    """Sanity: without the split, un-rounded inputs lose ~1e-3 (the MMA truncates)."""
    err = run_conv(2, 14, 14, 64, 128, 1, 1, 1, 0, raw_input=True)
    assert 1e-5 < err < 5e-3


@pytest.mark.gpu
@pytest.mark.parametrize("k,stride,pad,ceil,H", [(3, 1, 1, True, 14), (3, 2, 0, True, 112), (3, 2, 1, False, 56),
                                                (2, 2, 0, True, 14), (3, 2, 0, True, 28), (3, 2, 0, True, 13),
                                                (3, 1, 1, True, 7), (3, 2, 0, True, 15), (3, 1, 1, False, 9)])
def test_maxpool_in_executor_layers(k, stride, pad, ceil, H):
    """Max-pool shapes of GoogLeNet/ResNet-50 through a one-op network
    (the executor's own launch path) against the oracle."""
    from oracle.layers import maxpool_nhwc
    import ctypes as C
    from paper_2304_09961_b200._native import exec_lib, fptr
    lib = exec_lib()
    lib.bs_kernel_maxpool.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(1)
    n, c = 3, 64
    x = rng.standard_normal((n, H, H, c)).astype(np.float32)
    ref = maxpool_nhwc(x, k, stride, pad, ceil)
    out = np.zeros_like(ref)
    rc = lib.bs_kernel_maxpool(n, H, H, c, ref.shape[1], ref.shape[2], k, stride * 16 + pad, fptr(x), fptr(out))
    assert rc == 0
    assert np.array_equal(out, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("block", ["22", "24", "44"])
@pytest.mark.parametrize("H,ceil", [(28, True), (14, True), (10, False), (7, True), (9, False)])
def test_maxpool_stride1_tiles(block, H, ceil, monkeypatch):
    """Stride-1 3x3 pools with 2x2 / 2x4 / 4x4 output tiles per thread
    (BS_POOL_BLOCK), partial tiles at the right / bottom edges."""
    monkeypatch.setenv("BS_POOL_BLOCK", block)
    test_maxpool_in_executor_layers(3, 1, 1, ceil, H)


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if c["N"] > 128] + [
    dict(nimg=9, H=14, W=14, Cin=64, N=208, KH=3, KW=3, stride=1, pad=1)],
    ids=lambda c: "x".join(str(c[k]) for k in ("nimg", "H", "Cin", "N", "KH", "stride")))
@pytest.mark.parametrize("split", [1, 0])
def test_conv_wide_tiles(case, split, monkeypatch):
    """128 x 256 tiles (single TMEM accumulator), forced with BS_CONV_BN256=2."""
    monkeypatch.setenv("BS_CONV_BN256", "2")
    assert run_conv(**case, split=split) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    dict(nimg=3, H=28, W=28, Cin=64, N=192, KH=3, KW=3, stride=1, pad=1),
    dict(nimg=2, H=14, W=14, Cin=96, N=208, KH=3, KW=3, stride=1, pad=1),
    dict(nimg=5, H=7, W=7, Cin=256, N=384, KH=1, KW=1, stride=1, pad=0),
    dict(nimg=1, H=14, W=14, Cin=128, N=192, KH=3, KW=3, stride=1, pad=1),  # small M: split-K clusters
], ids=lambda c: f"b{c['nimg']}_N{c['N']}_k{c['KH']}")
@pytest.mark.parametrize("split", [0, 1])
def test_conv_192_wide_tiles(case, split, monkeypatch):
    # 128 x 192 tiles (two TMEM accumulators), forced
    monkeypatch.setenv("BS_CONV_BN192", "2")
    assert run_conv(**case, split=split, residual=True, relu=1) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    dict(nimg=2, H=14, W=14, Cin=160, N=320, KH=3, KW=3, stride=1, pad=1),
    dict(nimg=3, H=7, W=7, Cin=64, N=160, KH=1, KW=1, stride=1, pad=0),
    dict(nimg=1, H=14, W=14, Cin=96, N=480, KH=3, KW=3, stride=1, pad=1),  # split-K clusters
], ids=lambda c: f"b{c['nimg']}_N{c['N']}_k{c['KH']}")
def test_conv_160_wide_tiles(case, monkeypatch):
    # 128 x 160 tiles (two TMEM accumulators), forced
    monkeypatch.setenv("BS_CONV_BN160", "2")
    monkeypatch.setenv("BS_CONV_BN192", "0")
    assert run_conv(**case, split=1, residual=True, relu=1) < TOL
