"""PFM I/O (pfm.cpp:51-114) through the C ABI (host-only functions of libtsb.so, no GPU)
and the numpy oracle, pinned to the reference's tests/unit/test_pfm.cpp cases."""
import numpy as np
import pytest

from oracle import pfm as opfm


@pytest.fixture(scope="module")
def tsb():
    import paper_2505_05356_b200 as m
    return m


def _impls(tsb):
    return [("abi", tsb.write_pfm, tsb.read_pfm), ("oracle", opfm.write_pfm, opfm.read_pfm)]


def test_grayscale_round_trip_is_bit_exact(tsb, tmp_path):
    """test_pfm.cpp:28-51 (f32 values, a NaN; write -> read -> write reproduces the bytes)."""
    img = np.random.default_rng(3).uniform(-10, 10, (1, 5, 7)).astype(np.float32)
    img[0, 3, 2] = np.nan
    for name, wr, rd in _impls(tsb):
        p1, p2 = tmp_path / f"{name}_1ch.pfm", tmp_path / f"{name}_1ch_b.pfm"
        wr(p1, img)
        back = rd(p1)
        assert back.shape == img.shape
        assert np.array_equal(np.isnan(back), np.isnan(img))
        assert np.array_equal(back[~np.isnan(back)], img[~np.isnan(img)])
        wr(p2, back)
        assert p1.read_bytes() == p2.read_bytes()
    # the library and the oracle write the same bytes
    assert (tmp_path / "abi_1ch.pfm").read_bytes() == (tmp_path / "oracle_1ch.pfm").read_bytes()


def test_three_channel_round_trip(tsb, tmp_path):
    """test_pfm.cpp:53-61: channels interleaved per pixel in the file, planar in memory."""
    img = (0.25 * np.arange(3 * 3 * 4) - 2).astype(np.float32).reshape(3, 3, 4)
    for name, wr, rd in _impls(tsb):
        p = tmp_path / f"{name}_3ch.pfm"
        wr(p, img)
        assert np.array_equal(rd(p), img)
    assert (tmp_path / "abi_3ch.pfm").read_bytes() == (tmp_path / "oracle_3ch.pfm").read_bytes()
    # the first written pixel is the bottom-left one, its three channels in order
    raw = np.frombuffer((tmp_path / "abi_3ch.pfm").read_bytes()[len(b"PF\n4 3\n-1.0\n"):], "<f4")
    assert np.array_equal(raw[:3], img[:, 2, 0])


def test_header_and_bottom_to_top_rows(tsb, tmp_path):
    """test_pfm.cpp:63-80."""
    img = np.array([[[1.0], [2.0]]], np.float32)  # (1, H=2, W=1): top 1, bottom 2
    p = tmp_path / "rows.pfm"
    tsb.write_pfm(p, img)
    b = p.read_bytes()
    header = b"Pf\n1 2\n-1.0\n"
    assert len(b) == len(header) + 8 and b[:len(header)] == header
    assert np.array_equal(np.frombuffer(b[len(header):], "<f4"), [2.0, 1.0])


def test_positive_scale_is_big_endian(tsb, tmp_path):
    """test_pfm.cpp:82-95; also a '#' comment in the header."""
    p = tmp_path / "be.pfm"
    p.write_bytes(b"Pf\n# comment line\n1 1\n1.0\n" + np.array([3.5], ">f4").tobytes())
    for _, _, rd in _impls(tsb):
        assert rd(p)[0, 0, 0] == 3.5


def test_malformed_files_are_rejected(tsb, tmp_path):
    """test_pfm.cpp:97-105 (+ truncated data, bad dimensions, 2-channel write)."""
    bad = tmp_path / "bad.pfm"
    bad.write_bytes(b"P6\n1 1\n255\nxxx")
    trunc = tmp_path / "trunc.pfm"
    trunc.write_bytes(b"Pf\n2 2\n-1.0\n" + np.zeros(3, "<f4").tobytes())
    dims = tmp_path / "dims.pfm"
    dims.write_bytes(b"Pf\n0 2\n-1.0\n")
    for _, wr, rd in _impls(tsb):
        for path, msg in ((bad, "bad magic"), (tmp_path / "missing.pfm", "cannot open"), (trunc, "truncated"),
                          (dims, "bad dimensions")):
            with pytest.raises(RuntimeError, match=msg):
                rd(path)
        with pytest.raises(RuntimeError, match="1- or 3-channel"):
            wr(tmp_path / "two.pfm", np.zeros((2, 2, 2), np.float32))


def test_quad_decode_matches_host_helper(tsb):
    """oracle quad_to_depth (tof.hpp:47-65) == the library's tsb_quad_to_depth per pixel."""
    rng = np.random.default_rng(4)
    q = rng.normal(size=(4, 50))
    q[:, 0] = [0.3, 0.1, 0.3, 0.1]  # both differences vanish -> NaN
    d = opfm.quad_to_depth(q, 30e6)
    for i in range(50):
        ref = tsb.quad_to_depth(*q[:, i], 30e6)
        assert (np.isnan(d[i]) and np.isnan(ref)) or abs(d[i] - ref) <= 4e-16 * abs(ref)  # atan2 ulp
