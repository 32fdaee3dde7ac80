"""The DeformNet oracle pinned to the reference's own tests (tests/unit/test_deform.cpp)."""
import numpy as np

from oracle import deform as od


def test_positional_encoding_values_and_derivative():
    """test_deform.cpp:13-35."""
    assert od.encoding_size(0) == 1 and od.encoding_size(4) == 9
    e = od.positional_encode(0.25, 3)
    ref = [0.25, np.sin(np.pi * .25), np.cos(np.pi * .25), np.sin(2 * np.pi * .25), np.cos(2 * np.pi * .25),
           np.sin(4 * np.pi * .25), np.cos(4 * np.pi * .25)]
    assert np.allclose(e, ref, rtol=1e-12, atol=1e-15)
    v, h = 0.37, 1e-6
    d = od.positional_encode_derivative(v, 3)
    fd = (od.positional_encode(v + h, 3) - od.positional_encode(v - h, 3)) / (2 * h)
    assert np.allclose(d, fd, rtol=1e-4, atol=1e-6)


def test_fresh_net_is_nearly_identity():
    """test_deform.cpp:37-59: layer count, input dim, tiny initial offsets, determinism."""
    cfg = od.DeformConfig(hidden_layers=2, width=32)
    net = od.DeformNet.init(cfg, 3)
    assert net.input_dim == 3 * od.encoding_size(cfg.l_x) + od.encoding_size(cfg.l_t)
    assert len(net.W) == cfg.hidden_layers + 1
    pos = np.random.default_rng(5).uniform(-1, 1, (20, 3))
    for t in (0.0, 0.31, 1.0):
        off = net.offsets(pos, t)
        assert off.shape == pos.shape and np.abs(off).max() < 1e-3
    net2 = od.DeformNet.init(cfg, 3)
    assert np.array_equal(net.offsets(pos, 0.5), net2.offsets(pos, 0.5))


def test_gradients_match_finite_differences():
    """test_deform.cpp:61-114: parameter and input-position gradients vs central differences."""
    cfg = od.DeformConfig(hidden_layers=2, width=6, l_x=2, l_t=2, final_std=0.05, coord_scale=2.0)
    net = od.DeformNet.init(cfg, 9)
    rng = np.random.default_rng(13)
    pos = rng.uniform(-1, 1, (5, 3))
    up = rng.uniform(-1, 1, (5, 3))
    t = 0.41
    _, cache = net.offsets(pos, t, with_cache=True)
    dW, db, d_pos = net.backward(cache, up)
    analytic = net.flat_grads(dW, db)
    theta = net.get_parameters()
    h = 1e-5
    obj = lambda: float((net.offsets(pos, t) * up).sum())
    for i in range(theta.size):
        tp = theta.copy()
        tp[i] += h
        net.set_parameters(tp)
        fp = obj()
        tp[i] -= 2 * h
        net.set_parameters(tp)
        fm = obj()
        fd = (fp - fm) / (2 * h)
        assert abs(analytic[i] - fd) <= 1e-4 * max(1.0, abs(fd))
    net.set_parameters(theta)
    for c in range(pos.shape[0]):
        for r in range(3):
            pp = pos.copy()
            pp[c, r] += h
            fp = float((net.offsets(pp, t) * up).sum())
            pp[c, r] -= 2 * h
            fm = float((net.offsets(pp, t) * up).sum())
            assert abs(d_pos[c, r] - (fp - fm) / (2 * h)) <= 1e-4 * max(1.0, abs((fp - fm) / (2 * h)))


def test_parameter_round_trip():
    """test_deform.cpp:116-156 (parameter part): set/get is exact; flat order W row-major then b."""
    cfg = od.DeformConfig(hidden_layers=3, width=10, l_x=4, l_t=6, coord_scale=5.0, final_std=0.02)
    net = od.DeformNet.init(cfg, 21)
    theta = np.random.default_rng(2).uniform(-0.5, 0.5, net.parameter_count)
    net.set_parameters(theta)
    assert np.array_equal(net.get_parameters(), theta)
    assert np.array_equal(net.W[0].ravel(), theta[:net.W[0].size])


def test_interp_positions():
    """test_deform.cpp:158-172."""
    a = np.array([[0, 1, 2], [3, 4, 5]], float).T
    b = np.array([[10, -1, 0], [3, 8, 7]], float).T
    assert np.array_equal(od.interp_positions(a, b, 2.0, 3.0, 2.0), a)
    assert np.array_equal(od.interp_positions(a, b, 2.0, 3.0, 3.0), b)
    assert np.allclose(od.interp_positions(a, b, 2.0, 3.0, 2.5), 0.5 * (a + b), rtol=1e-15)
