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
    r = ctx.selftest_affine(2, 30, 64, 64)
    assert r["err_umma"] == -1.0 and r["err_simt"] < 2e-6
