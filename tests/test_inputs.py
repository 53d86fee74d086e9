"""Input formats (S0 ingest, no GPU): the packed 12-bit ADC byte format produced by
synth.generate.pack12 round-trips through an independent bit-level unpacking, for
the full 12-bit code range and random streams."""
import numpy as np

import pytest

from synth.generate import pack12


def _unpack_ref(b):
    """bit-by-bit reference: sample k occupies bits [12k, 12k+12) of the little-endian byte stream"""
    bits = np.unpackbits(np.asarray(b, dtype=np.uint8), bitorder="little")
    n = bits.size // 12
    v = bits[:12 * n].reshape(n, 12).astype(np.int64) @ (1 << np.arange(12))
    return np.where(v >= 2048, v - 4096, v).astype(np.int16)


def test_pack12_full_range_round_trip():
    c = np.arange(-2048, 2048, dtype=np.int16)
    p = pack12(c)
    assert p.dtype == np.uint8 and p.size == c.size * 3 // 2
    assert np.array_equal(_unpack_ref(p), c)


def test_pack12_random_stream_and_layout():
    rng = np.random.default_rng(3)
    c = rng.integers(-2048, 2048, 10_000).astype(np.int16)
    assert np.array_equal(_unpack_ref(pack12(c)), c)
    # documented byte layout of one pair (include/kk_rx.h): c0 = 0xABC (-1348), c1 = 0x123
    p = pack12(np.array([0xABC - 4096, 0x123], dtype=np.int16))
    assert list(p) == [0xBC, 0x3A, 0x12]


def test_hermgauss_exactness():
    """kk_hermgauss (host, Golub-Welsch): the n-node rule integrates t^(2j) e^(-t^2)
    exactly (= Gamma(j + 1/2)) for 2j <= 2n - 1, odd moments vanish; nodes/weights equal
    numpy's rule."""
    import math
    from paper_2108_07004_b200 import hermgauss
    for n in (1, 2, 6, 10, 20):
        t, w = hermgauss(n)
        assert np.all(np.diff(t) > 0) and np.all(w > 0)
        for j in range(n):
            assert abs(np.sum(w * t ** (2 * j)) - math.gamma(j + 0.5)) <= 1e-12 * max(1.0, math.gamma(j + 0.5))
            assert abs(np.sum(w * t ** (2 * j + 1))) <= 1e-11 * max(1.0, math.gamma(j + 1.0))
        t0, w0 = np.polynomial.hermite.hermgauss(n)
        assert np.max(np.abs(t - t0)) < 1e-12 and np.max(np.abs(w - w0)) < 1e-12


def test_gs_tool_writes_loadable_binary_labels(tmp_path):
    """tools/gs_optimize_gpu.write_constellation (the GPU optimiser's --write output) writes
    labels as log2(M)-bit binary strings that synth.generate.load_constellation_file reads
    back exactly (round-1 ADVICE: it wrote decimal labels the loader parsed as binary)."""
    import importlib.util
    import os
    import numpy as np
    from synth.generate import load_constellation, load_constellation_file
    spec = importlib.util.spec_from_file_location(
        "gs_optimize_gpu", os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools", "gs_optimize_gpu.py"))
    gs = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gs)
    rng = np.random.default_rng(5)
    for name in ("QAM8", "GS128"):
        p, l = load_constellation(name)
        perm = rng.permutation(len(p))
        path = tmp_path / f"{name}.txt"
        gs.write_constellation(str(path), p, l[perm], "round trip\nsecond header line")
        p2, l2 = load_constellation_file(str(path))
        assert np.array_equal(l2, l[perm])
        assert np.max(np.abs(p2 - p)) < 1e-15
    with pytest.raises(AssertionError):
        gs.write_constellation(str(tmp_path / "bad.txt"), p[:3], [0, 1, 1], "not a bijection")
