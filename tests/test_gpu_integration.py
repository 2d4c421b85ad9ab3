"""The simdet::gpu shim (integration/simdet_gpu.cpp -- the reference-side
binding of INTEGRATION.md §2) on reference Tensors, against the reference
engine's own CPU functions (oracle/_ref) on identical inputs: conv2d and its
Tape backward rule, syncbn_forward/backward (group == nullptr, incl. the 2C+1
aggregation sums), iabn_forward/backward, and apply_sgd (bitwise vs
sgd_step_master at scale 1, K 1) -- plus the reference exception taxonomy
(NonInvertibleError, DegenerateBatchError) raised through the shim."""
import numpy as np
import pytest

from oracle import p
from tests import shim
from tests.util import assert_close

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not shim.available(), reason="shim not built")]


@pytest.mark.parametrize("fp16", [0, 1])
def test_shim_conv2d_and_backward(ref, fp16):
    lb = shim.lib()
    rng = np.random.default_rng(7 + fp16)
    N, C, H, W, O, k, s, pd = 2, 32, 20, 17, 64, 3, 2, 1
    x = rng.standard_normal((N, C, H, W)).astype(np.float32)
    w = (0.1 * rng.standard_normal((O, C, k, k))).astype(np.float32)
    if fp16:
        x, w = x.astype(np.float16).astype(np.float32), w.astype(np.float16).astype(np.float32)
    Ho, Wo = (H + 2 * pd - k) // s + 1, (W + 2 * pd - k) // s + 1
    y, y_ref = np.zeros((N, O, Ho, Wo), np.float32), np.zeros((N, O, Ho, Wo), np.float32)
    assert lb.shim_conv2d(p(x), N, C, H, W, p(w), O, k, k, s, pd, fp16, p(y)) == 0, lb.shim_last_error()
    assert ref.ref_conv2d(p(x), N, C, H, W, p(w), O, k, k, s, pd, fp16, p(y_ref)) == 0
    tol = 1e-2 if fp16 else 1e-5
    assert_close(y, y_ref, tol, "shim conv2d")
    dy = rng.standard_normal(y.shape).astype(np.float32)
    dx, dk = np.zeros_like(x), np.zeros_like(w)
    dx_r, dk_r = np.zeros_like(x), np.zeros_like(w)
    assert lb.shim_conv2d_backward(p(x), N, C, H, W, p(w), O, k, k, s, pd, fp16, p(dy), p(dx), p(dk)) == 0
    assert ref.ref_conv2d_backward(p(x), N, C, H, W, p(w), O, k, k, s, pd, fp16, p(dy), p(dx_r), p(dk_r)) == 0
    assert_close(dx, dx_r, tol, "shim conv2d dx")
    assert_close(dk, dk_r, tol, "shim conv2d dk")


@pytest.mark.parametrize("fp16", [0, 1])
def test_shim_batchnorm(ref, fp16):
    lb = shim.lib()
    rng = np.random.default_rng(11 + fp16)
    N, C, H, W = 2, 64, 9, 13
    x = (2 + 3 * rng.standard_normal((N, C, H, W))).astype(np.float32)
    if fp16:
        x = x.astype(np.float16).astype(np.float32)
    g = rng.uniform(0.5, 1.5, C).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, C).astype(np.float32)
    y, mu, inv = np.zeros_like(x), np.zeros(C, np.float32), np.zeros(C, np.float32)
    sm, sq, cnt = np.zeros(C, np.float32), np.zeros(C, np.float32), np.zeros(1, np.int64)
    assert lb.shim_bn_forward(p(x), N, C, H, W, p(g), p(b), 1e-5, fp16, p(y), p(mu), p(inv), p(sm), p(sq), p(cnt)) == 0
    y_r, mu_r, inv_r = np.zeros_like(x), np.zeros(C, np.float32), np.zeros(C, np.float32)
    assert ref.ref_bn_forward(p(x), N, C, H, W, p(g), p(b), 1e-5, fp16, p(y_r), p(mu_r), p(inv_r)) == 0
    assert cnt[0] == N * H * W
    np.testing.assert_allclose(sm, x.transpose(1, 0, 2, 3).reshape(C, -1).sum(1, dtype=np.float64), rtol=1e-6)
    np.testing.assert_allclose(mu, mu_r, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(inv, inv_r, rtol=1e-6)
    assert_close(y, y_r, 1e-2 if fp16 else 1e-6, "shim bn fwd")
    dy = rng.standard_normal(x.shape).astype(np.float32)
    dx, dg, db = np.zeros_like(x), np.zeros(C, np.float32), np.zeros(C, np.float32)
    dx_r, dg_r, db_r = np.zeros_like(x), np.zeros(C, np.float32), np.zeros(C, np.float32)
    assert lb.shim_bn_backward(p(dy), p(x), N, C, H, W, p(g), p(mu_r), p(inv_r), fp16, p(dx), p(dg), p(db)) == 0
    assert ref.ref_bn_backward(p(dy), p(x), N, C, H, W, p(g), p(mu_r), p(inv_r), fp16, p(dx_r), p(dg_r), p(db_r)) == 0
    tol = 1e-2 if fp16 else 1e-5
    assert_close(dx, dx_r, tol, "shim bn dx")
    assert_close(dg, dg_r, tol, "shim bn dgamma")
    assert_close(db, db_r, tol, "shim bn dbeta")


@pytest.mark.parametrize("fp16", [0, 1])
def test_shim_iabn_and_errors(ref, fp16):
    lb = shim.lib()
    rng = np.random.default_rng(13 + fp16)
    N, C, H, W = 2, 128, 7, 11
    x = rng.standard_normal((N, C, H, W)).astype(np.float32)
    if fp16:
        x = x.astype(np.float16).astype(np.float32)
    g = rng.uniform(0.5, 1.5, C).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, C).astype(np.float32)
    y, mu, inv = np.zeros_like(x), np.zeros(C, np.float32), np.zeros(C, np.float32)
    assert lb.shim_iabn_forward(p(x), N, C, H, W, p(g), p(b), 1e-5, 0.1, fp16, p(y), p(mu), p(inv)) == 0
    y_r, mu_r, inv_r = np.zeros_like(x), np.zeros(C, np.float32), np.zeros(C, np.float32)
    assert ref.ref_iabn_forward(p(x), N, C, H, W, p(g), p(b), 1e-5, 0.1, fp16, p(y_r), p(mu_r), p(inv_r)) == 0
    tol = 1e-2 if fp16 else 1e-5
    assert_close(y, y_r, tol, "shim iabn fwd")
    dy = rng.standard_normal(x.shape).astype(np.float32)
    dx, dg, db = np.zeros_like(x), np.zeros(C, np.float32), np.zeros(C, np.float32)
    dx_r, dg_r, db_r = np.zeros_like(x), np.zeros(C, np.float32), np.zeros(C, np.float32)
    assert lb.shim_iabn_backward(p(dy), p(y_r), N, C, H, W, p(g), p(b), p(mu_r), p(inv_r), 1e-5, 0.1, fp16, p(dx),
                                 p(dg), p(db)) == 0
    assert ref.ref_iabn_backward(p(dy), p(y_r), N, C, H, W, p(g), p(b), p(mu_r), p(inv_r), 1e-5, 0.1, fp16, p(dx_r),
                                 p(dg_r), p(db_r)) == 0
    assert_close(dx, dx_r, tol, "shim iabn dx")
    assert_close(dg, dg_r, tol, "shim iabn dgamma")
    assert_close(db, db_r, tol, "shim iabn dbeta")
    # the reference's contract errors through the shim (src/memopt.cpp:229-235)
    g0 = g.copy()
    g0[5] = 0.0
    assert lb.shim_iabn_forward(p(x), N, C, H, W, p(g0), p(b), 1e-5, 0.1, fp16, p(y), p(mu), p(inv)) == 4
    assert lb.shim_iabn_forward(p(x), N, C, H, W, p(g), p(b), 1e-5, 0.0, fp16, p(y), p(mu), p(inv)) == 4
    x1 = np.ascontiguousarray(x[:1, :, :1, :1])
    assert lb.shim_iabn_forward(p(x1), 1, C, 1, 1, p(g), p(b), 1e-5, 0.1, fp16, p(y), p(mu), p(inv)) == 3


def test_shim_apply_sgd_bitwise(ref):
    lb = shim.lib()
    rng = np.random.default_rng(17)
    n = 100_003
    w = rng.standard_normal(n).astype(np.float32)
    v = (0.1 * rng.standard_normal(n)).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    w_r, v_r = w.copy(), v.copy()
    sk = np.zeros(1, np.int32)
    assert lb.shim_apply_sgd(p(w), p(v), p(g), n, 0.01, 0.9, 1.0, 1, p(sk)) == 0 and sk[0] == 0
    assert ref.ref_sgd_step_master(p(w_r), p(v_r), p(g), n, 0.01, 0.9) == 0
    assert np.array_equal(w.view(np.uint32), w_r.view(np.uint32))
    assert np.array_equal(v.view(np.uint32), v_r.view(np.uint32))
    g[77] = np.inf
    w0 = w.copy()
    assert lb.shim_apply_sgd(p(w), p(v), p(g), n, 0.01, 0.9, 1.0, 1, p(sk)) == 0 and sk[0] == 1
    assert np.array_equal(w, w0)
