"""Pins of the oracle's HDC encoder / quantisers (not gpu)."""
import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import hdc, nt


def test_encode_raw_matches_loops():
    rng = np.random.default_rng(0)
    P = (2 * rng.integers(0, 2, size=(9, 13)) - 1).astype(np.int8)
    X = rng.integers(-128, 128, size=(5, 13)).astype(np.int8)
    acc = hdc.encode_raw(P, X, 7)
    for d in range(7):
        for q in range(5):
            assert acc[d, q] == sum(int(P[d, f]) * int(X[q, f]) for f in range(13))
    Xu = rng.integers(0, 256, size=(5, 13)).astype(np.uint8)
    accu = hdc.encode_raw(P, Xu, 9)
    assert accu[3, 2] == sum(int(P[3, f]) * int(Xu[2, f]) for f in range(13))


def test_quantise_queries_hand_examples():
    acc = np.array([[5, 6, -5, -6, 2, -2, 100, -100]], dtype=np.int64)
    h = hdc.quantise_queries(acc, 2, 3)     # qmax 3, floor((acc+2)/4)
    assert h.tolist() == [[1, 2, -1, -1, 1, 0, 3, -3]]
    assert hdc.quantise_queries(np.array([[4, -9]]), 0, 3).tolist() == [[3, -3]]


def test_quantise_classes_round_half_away():
    v = np.array([[3, -3, 1, -1, 0], [2, -2, 4, 1, 0]], dtype=np.int64)
    C = hdc.quantise_classes(v, 4)           # cmax 7
    assert C[0].tolist() == [7, -7, 2, -2, 0]
    assert C[1].tolist() == [4, -4, 7, 2, 0]  # 3.5 -> 4, -3.5 -> -4, 1.75 -> 2
    assert hdc.quantise_classes(np.zeros((1, 3), np.int64), 4).tolist() == [[0, 0, 0]]


@pytest.mark.parametrize("name,Q", [("c1", 3), ("c2", 5), ("c3", 6), ("c4", 8)])
def test_query_width_no_wrap(name, Q):
    cfg = inp.CONFIGS[name]
    t = nt.plaintext_modulus(cfg.t_bits, cfg.log2N, cfg.t_fixed)
    got = hdc.choose_Qbits(cfg.D_live, cfg.Cbits, t)
    assert got == Q
    cmax = hdc.qmax_of(cfg.Cbits)
    assert cfg.D_live * hdc.qmax_of(got) * cmax <= (t - 1) // 2
    if got < 8:
        assert cfg.D_live * hdc.qmax_of(got + 1) * cmax > (t - 1) // 2


def test_calibrate_shift():
    acc = np.array([[0, 37, -50]], dtype=np.int64)
    s = hdc.calibrate_shift(acc, 3)         # qmax 3: 3*2^4=48 < 50 <= 96
    assert s == 5
    assert hdc.calibrate_shift(np.array([[3]]), 3) == 0


def test_bundle_and_argmax():
    acc = np.array([[1, 2, 3, 4], [5, 6, 7, 8]], dtype=np.int64)
    y = np.array([0, 1, 0, 1])
    assert hdc.bundle(acc, y, 2).tolist() == [[4, 12], [6, 14]]
    S = np.array([[1, 3, 3], [5, 5, 0], [0, 0, 0]])
    assert hdc.argmax_lowest(S).tolist() == [1, 0, 0]     # ties -> lowest index
