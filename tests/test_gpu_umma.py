"""tcgen05 (UMMA) 3xTF32 bound GEMM: FP32-class accuracy against an f64 reference, on the
shapes of the BASELINE configs' affines (M = O, K = C, N = D) and edge tilings."""
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [
    # rows, C, O, D
    (2, 128, 128, 128),    # single tile, BN=128 path
    (3, 64, 256, 256),     # two k-blocks, BN=256 path
    (4, 256, 768, 512),    # c3 QKV
    (2, 512, 256, 512),    # c3 W2
    (2, 128, 384, 128),    # c2 QKV
    (1, 768, 256, 1536),   # c5-like N
    (5, 96, 128, 384),     # odd tile counts (3 k-blocks, 3 N tiles of 128)
    (64, 64, 192, 64),     # c1 QKV: D = 64, token rows folded in pairs into the 128 TMEM lanes
    (32, 128, 64, 64),     # c1 W2 (K = 128): folded
]


@pytest.mark.parametrize("rows,c,o,d", SHAPES)
def test_umma_affine_matches_f64(ctx, rows, c, o, d):
    r = ctx.selftest_affine(rows, c, o, d, seed=rows * 7 + c)
    assert r["err_simt"] < 2e-6, r
    assert r["err_umma"] >= 0, "shape unexpectedly not tcgen05-eligible"
    # 3xTF32 on tcgen05: measured 2-4e-6 of max|Y| for K = 256..768 (the tensor core's fp32
    # accumulation is not round-to-nearest); 1xTF32 would be ~1e-3.  Bound: 1e-5.
    assert r["err_umma"] < 1e-5, r


def test_umma_ineligible_shape_reports(ctx):
    r = ctx.selftest_affine(2, 30, 64, 64)  # C % 32 != 0
    assert r["err_umma"] == -1.0 and r["err_simt"] < 2e-6
    r = ctx.selftest_affine(3, 64, 64, 64)  # D = 64 with an odd number of rows cannot fold
    assert r["err_umma"] == -1.0


def test_umma_bias_compensated(ctx):
    """The epilogue's truncation compensation leaves the tcgen05 planes unbiased: the median
    signed relative error of both planes stays well below the uncompensated 2-3e-6."""
    for c in (256, 512):
        r = ctx.selftest_affine(32, c, 256, 256, seed=c)
        assert abs(r["bias_umma_centre"]) < 1e-6 and abs(r["bias_umma_radius"]) < 1e-6, r
