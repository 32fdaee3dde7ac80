"""The image-loss oracle pinned to the reference's own tests (tests/unit/test_losses.cpp)."""
import numpy as np

from oracle import losses as ol


def rand_img(w, h, c, seed):
    return np.random.default_rng(seed).uniform(0, 1, (c, h, w))


def test_window_is_normalised_gaussian():
    w = ol.window1d()
    assert w.size == 11 and abs(w.sum() - 1) < 1e-15 and np.argmax(w) == 5 and np.allclose(w, w[::-1])


def test_ssim_of_identical_images_is_one():
    """test_losses.cpp:39-44."""
    a = rand_img(16, 12, 3, 5)
    assert abs(ol.ssim(a, a) - 1.0) < 1e-12
    assert ol.ssim(a, rand_img(16, 12, 3, 6)) < 1.0


def test_ssim_gradient_matches_finite_differences():
    """test_losses.cpp:46-62."""
    pred, target = rand_img(8, 8, 1, 7), rand_img(8, 8, 1, 8)
    _, g = ol.ssim(pred, target, True)
    h = 1e-6
    for i in range(pred.size):
        p = pred.copy().ravel()
        p[i] += h
        fp = ol.ssim(p.reshape(pred.shape), target)
        p[i] -= 2 * h
        fm = ol.ssim(p.reshape(pred.shape), target)
        fd = (fp - fm) / (2 * h)
        assert abs(g.ravel()[i] - fd) <= 1e-4 * max(abs(fd), 0.01)


def test_image_loss_blends_mse_and_ssim():
    """test_losses.cpp:64-87."""
    a, b = rand_img(12, 9, 2, 9), rand_img(12, 9, 2, 10)
    assert abs(ol.image_loss(a, a, 0.2)) < 1e-12
    assert np.isclose(ol.image_loss(a, b, 0.0), ol.mse(a, b), rtol=1e-12)
    assert np.isclose(ol.image_loss(a, b, 1.0), 1.0 - ol.ssim(a, b), rtol=1e-12)
    assert np.isclose(ol.image_loss(a, b, 0.2), 0.8 * ol.mse(a, b) + 0.2 * (1.0 - ol.ssim(a, b)), rtol=1e-12)
    pred, target = rand_img(8, 8, 1, 11), rand_img(8, 8, 1, 12)
    _, g = ol.image_loss(pred, target, 0.2, True)
    h = 1e-6
    for i in range(0, pred.size, 7):
        p = pred.copy().ravel()
        p[i] += h
        fp = ol.image_loss(p.reshape(pred.shape), target, 0.2)
        p[i] -= 2 * h
        fm = ol.image_loss(p.reshape(pred.shape), target, 0.2)
        fd = (fp - fm) / (2 * h)
        assert abs(g.ravel()[i] - fd) <= 1e-4 * max(abs(fd), 0.01)
