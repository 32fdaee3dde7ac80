"""DeformNet on the B200 tensor cores: the tcgen05 GEMM
(kind::tf32, 3xTF32 split) against fp64 numpy, then the network against the oracle
restatement of deform.cpp."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tsb():
    import paper_2505_05356_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(tsb):
    return tsb.Context(0)


def gemm(tsb, ctx, A, a_m, a_k, B, b_n, b_k, M, N, K, slices=1, bias=None, relu=0, mask=None):
    out = np.zeros((M, N), np.float32)
    f = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)
    A, B, bias, mask = f(A), f(B), f(bias), f(mask)
    p = lambda a: None if a is None else a.ctypes.data
    tsb._abi.check(tsb._abi.lib().tsb_debug_gemm(ctx.handle, M, N, K, slices, p(A), a_m, a_k, p(B), b_n, b_k,
                                                 p(bias), relu, p(mask), out.ctypes.data))
    return out


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (300, 128, 84), (257, 3, 128), (1000, 64, 200), (77, 16, 8)])
def test_gemm_row_major(tsb, ctx, M, N, K):
    rng = np.random.default_rng(M + N + K)
    A = rng.normal(size=(M, K)).astype(np.float32)
    W = rng.normal(size=(N, K)).astype(np.float32)
    bias = rng.normal(size=N).astype(np.float32)
    ref = A.astype(np.float64) @ W.astype(np.float64).T + bias
    got = gemm(tsb, ctx, A, K, 1, W, K, 1, M, N, K, bias=bias)
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 2e-6 * scale * np.sqrt(K), np.abs(got - ref).max() / scale
    relu = gemm(tsb, ctx, A, K, 1, W, K, 1, M, N, K, bias=bias, relu=1)
    assert np.abs(relu - np.maximum(ref, 0)).max() <= 2e-6 * scale * np.sqrt(K)


def test_gemm_transposed_operands_split_k_and_mask(tsb, ctx):
    """dW = delta^T H over many rows (both operands read transposed, split over K slices),
    and d_below = delta W gated by a ReLU mask."""
    rng = np.random.default_rng(7)
    n, o, k = 2000, 96, 112
    delta = rng.normal(size=(n, o)).astype(np.float32)
    H = rng.normal(size=(n, k)).astype(np.float32)
    # D[m=o][j=k] = sum_n delta[n][o] H[n][k]: A(m, kk) = delta[kk*o + m], B(j, kk) = H[kk*k + j]
    got = gemm(tsb, ctx, delta, 1, o, H, 1, k, o, k, n, slices=7)
    ref = delta.astype(np.float64).T @ H.astype(np.float64)
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()
    W = rng.normal(size=(o, k)).astype(np.float32)
    mask = (rng.random((n, k)) > 0.5).astype(np.float32)
    # d_below[n][j] = sum_o delta[n][o] W[o][j]: B(j, oo) = W[oo*k + j]
    got2 = gemm(tsb, ctx, delta, o, 1, W, 1, k, n, k, o, mask=mask)
    ref2 = (delta.astype(np.float64) @ W.astype(np.float64)) * mask
    assert np.abs(got2 - ref2).max() <= 1e-5 * np.abs(ref2).max()


@pytest.mark.parametrize("n,slices", [(5000, 7), (131, 1)])
def test_gemm_bulk_copied_transposed_operands(tsb, ctx, n, slices):
    """Full-width 128-column operands read transposed (dW of a hidden layer): the chunks are
    contiguous row runs moved by TMA bulk copies, partial last chunks zero-padded on split."""
    rng = np.random.default_rng(11)
    delta = rng.normal(size=(n, 128)).astype(np.float32)
    H = rng.normal(size=(n, 128)).astype(np.float32)
    got = gemm(tsb, ctx, delta, 1, 128, H, 1, 128, 128, 128, n, slices=slices)
    ref = delta.astype(np.float64).T @ H.astype(np.float64)
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()


@pytest.mark.parametrize("N,K", [(128, 128), (84, 128), (128, 3), (32, 64), (16, 40)])
def test_gemm_many_tiles_resident_weights(tsb, ctx, N, K):
    """delta W over more row tiles than CTAs (weights resident; the warp-specialised kernel:
    the epilogue drains one TMEM accumulator while the next tile fills the other), with and
    without a ReLU gate, partial column groups included."""
    rng = np.random.default_rng(N * 1000 + K)
    n = 148 * 128 * 2 + 777
    delta = rng.normal(size=(n, K)).astype(np.float32)
    W = rng.normal(size=(K, N)).astype(np.float32)
    ref = delta.astype(np.float64) @ W.astype(np.float64)
    tol = 2e-6 * np.abs(ref).max() * np.sqrt(K)
    got = gemm(tsb, ctx, delta, K, 1, W, 1, N, n, N, K)
    assert np.abs(got - ref).max() <= tol
    mask = (rng.random((n, N)) > 0.5).astype(np.float32)
    got2 = gemm(tsb, ctx, delta, K, 1, W, 1, N, n, N, K, mask=mask)
    assert np.abs(got2 - ref * mask).max() <= tol


def _nets(tsb, ctx, cfg, seed, n=3000):
    from oracle import deform as od
    onet = od.DeformNet.init(cfg, seed)
    # scale the tiny default output layer up so offsets and gradients exercise every layer
    rng = np.random.default_rng(seed + 1)
    onet.W[-1] = 0.05 * rng.normal(size=onet.W[-1].shape)
    for b in onet.b:
        b[:] = 0.01 * rng.normal(size=b.shape)
    theta = onet.get_parameters().astype(np.float32)
    onet.set_parameters(theta.astype(np.float64))  # both sides see the same fp32 values
    gnet = tsb.DeformNet(ctx, cfg.hidden_layers, cfg.width, cfg.l_x, cfg.l_t, cfg.coord_scale)
    gnet.set_parameters(theta)
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    return onet, gnet, pos, rng


def _rel(a, b, floor):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor * np.abs(b).max()))


def _check(got, ref, rel_tol, name=""):
    """Entry-wise relative error under a floor of 1e-2 x max|ref| (the offsets and
    gradients are sums of 64-128 signed products that cancel to ~1e-6 of their terms;
    3xTF32 resolves them to ~1e-7 of the buffer maximum, not of themselves) and
    normwise error (max abs / max|ref|) below rel_tol / 10."""
    r = _rel(got, ref, 1e-2)
    nw = np.abs(np.asarray(got, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30)
    assert r < rel_tol and nw < rel_tol / 10, (name, r, nw)


@pytest.mark.parametrize("layers,width,lx,lt,scale", [(4, 128, 10, 10, 1.0), (2, 32, 4, 6, 2.5), (0, 16, 2, 2, 1.0)])
def test_deform_forward_backward_vs_oracle(tsb, ctx, layers, width, lx, lt, scale):
    """deform.cpp:80-159 on the tensor cores vs the fp64 restatement: offsets (1e-4 rel),
    dW/db and d(position) (1e-3 rel, floor 1e-4 x max per quantity)."""
    from oracle import deform as od
    cfg = od.DeformConfig(hidden_layers=layers, width=width, l_x=lx, l_t=lt, coord_scale=scale)
    onet, gnet, pos, rng = _nets(tsb, ctx, cfg, 11 + layers)
    t = 0.37
    ref, cache = onet.offsets(pos.astype(np.float64), t, with_cache=True)
    got = gnet.offsets(pos, t, slot=1)
    _check(got, ref, 1e-4, "offsets")
    up = rng.normal(size=pos.shape).astype(np.float32)
    dW, db, dpos = onet.backward(cache, up.astype(np.float64))
    gnet.zero_grads()
    gdpos = gnet.backward(up, slot=1)
    gflat, oflat = gnet.grads(), onet.flat_grads(dW, db)
    k = 0
    for w, b in zip(dW, db):
        for part in (w.ravel(), b):
            _check(gflat[k:k + part.size], part, 1e-3, f"param block at {k}")
            k += part.size
    _check(gdpos, dpos, 1e-3, "d_position")
    # gradients accumulate (Grads are summed across renders, trainer.cpp:325-335)
    gnet.backward(up, slot=1, want_positions=False)
    _check(gnet.grads(), 2 * oflat, 1e-3, "accumulated")


def test_deform_position_gradient_many_tiles(tsb, ctx):
    """d(position) at 40k points (more row tiles than CTAs: the encoding chain runs fused
    in the input-gradient GEMM's epilogue, l_x = 10), then accumulated into a second call."""
    from oracle import deform as od
    cfg = od.DeformConfig()
    onet, gnet, pos, rng = _nets(tsb, ctx, cfg, 23, n=40_000)
    t = 0.61
    ref, cache = onet.offsets(pos.astype(np.float64), t, with_cache=True)
    got = gnet.offsets(pos, t, slot=1)  # (entry-wise offsets are checked above; normwise here)
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()
    up = rng.normal(size=pos.shape).astype(np.float32)
    # the oracle backward through the GPU's ReLU gates (see test_deform_large_batch_and_adam)
    gates = [gnet.debug_activation(lv, pos.shape[0], slot=1) > 0 for lv in range(cfg.hidden_layers)]
    _, _, dpos = onet.backward(cache, up.astype(np.float64), gates=gates)
    gnet.zero_grads()
    gdpos = gnet.backward(up, slot=1)
    _check(gdpos, dpos, 1e-3, "d_position")


def test_deform_large_batch_and_adam(tsb, ctx):
    """200k points (many row tiles and weight-gradient slices), then one Adam step on the
    network parameters equals the reference AdamState::step (trainer.cpp:18-31)."""
    from oracle import deform as od
    from oracle import oracle as orc
    cfg = od.DeformConfig()
    onet, gnet, pos, rng = _nets(tsb, ctx, cfg, 5, n=200_000)
    t = 0.8
    ref, cache = onet.offsets(pos.astype(np.float64), t, with_cache=True)
    _check(gnet.offsets(pos, t), ref, 1e-4, "offsets")
    up = rng.normal(size=pos.shape).astype(np.float32)
    gnet.zero_grads()
    gnet.backward(up, want_positions=False)
    g = gnet.grads()
    # ReLU gates whose fp64 pre-activation lies within the 3xTF32 error (~1e-6 of the
    # layer's scale) of zero can open differently from the reference (the MLP analogue of
    # the raster's threshold decisions; there is no fp64 fix-up for it).  The arithmetic is
    # checked against the oracle backward taken through the GPU's own gates at 1e-3; the
    # end-to-end gradient with the reference's gates normwise at 1e-3.
    gates = [gnet.debug_activation(lv, pos.shape[0]) > 0 for lv in range(cfg.hidden_layers)]
    flips = sum(int((gt != (h > 0)).sum()) for gt, h in zip(gates, cache.h))
    assert flips <= 1e-5 * pos.shape[0] * cfg.width * cfg.hidden_layers, flips
    dW, db, _ = onet.backward(cache, up.astype(np.float64), want_positions=False, gates=gates)
    _check(g, onet.flat_grads(dW, db), 1e-3, "grads (GPU gates)")
    dW, db, _ = onet.backward(cache, up.astype(np.float64), want_positions=False)
    ref = onet.flat_grads(dW, db)
    assert np.abs(g - ref).max() <= 1e-3 * np.abs(ref).max()
    before = gnet.get_parameters().astype(np.float64)
    gnet.adam_step(1e-3)
    after = gnet.get_parameters().astype(np.float64)
    p, m, v = before.copy(), np.zeros_like(before), np.zeros_like(before)
    orc.adam_step(p, g.astype(np.float64), m, v, 1, 1e-3)
    assert np.abs((after - before) - (p - before)).max() <= 1e-6


def test_deform_drives_scene_keyframes(tsb, ctx):
    """Scene coupling (trainer.cpp:262-279, 325-335): the network's offsets at two tick
    times become keyframes 0/1; rendering at w and back-propagating gives the same
    position gradient as the oracle chain through both ticks."""
    from oracle import deform as od
    from paper_2505_05356_b200 import synthetic
    from helpers import gpu_scene
    cfg = od.DeformConfig(hidden_layers=2, width=64, l_x=6, l_t=4)
    onet, gnet, _, rng = _nets(tsb, ctx, cfg, 3)
    g = synthetic.gaussians(3000, 4, n_keyframes=2)
    scene = gpu_scene(tsb, ctx, g, tsb.ToFConfig(30e6))
    ti, tip1 = 0.25, 0.5
    gnet.scene_offsets(scene, 0, ti, slot=0)
    gnet.scene_offsets(scene, 1, tip1, slot=2)
    prm = scene.get_params()
    pos64 = g.position.astype(np.float64)
    _check(prm["motion"][0], onet.offsets(pos64, ti), 1e-4, "keyframe 0")
    _check(prm["motion"][1], onet.offsets(pos64, tip1), 1e-4, "keyframe 1")
    assert np.array_equal(prm["position"], g.position)
    # a render at w = 0.5 and an arbitrary upstream, then the network backward for both ticks
    cam = synthetic.camera(160, 120, 140.0)
    rp = tsb.RenderPass(ctx).prepare(scene, cam, tsb.RenderOptions(), (0, 0.5)).forward()
    up = rng.normal(size=(4, 120, 160)).astype(np.float32) * 1e-2
    scene.zero_grads()
    rp.backward(up)
    before = scene.grads()
    gnet.zero_grads()
    gnet.scene_backward(scene, 0, slot=0)
    gnet.scene_backward(scene, 1, slot=2)
    after = scene.grads()
    # the network adds d(offsets)/d(position) of each tick's keyframe gradient
    _, ci = onet.offsets(pos64, ti, with_cache=True)
    _, cj = onet.offsets(pos64, tip1, with_cache=True)
    _, _, di = onet.backward(ci, before["d_motion"][0].astype(np.float64))
    _, _, dj = onet.backward(cj, before["d_motion"][1].astype(np.float64))
    _check(after["d_position"].astype(np.float64) - before["d_position"], di + dj, 1e-3, "d_position")
