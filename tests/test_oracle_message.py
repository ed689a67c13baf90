"""Pins of the scores-message oracle (NEXT #4; not gpu): a hand-computed bit layout,
the size formula, roundtrip, and the saving against 64-bit words at c2-c4."""
import numpy as np

import ephdc_inputs as inp
from oracle import message, nt


def test_hand_computed_layout():
    # q = 5 (3 bits), N = 8, values 1 2 3 4 0 1 2 3 at bit offsets 0, 3, ..., 21 (LSB first):
    # byte0 = bits {0, 4, 6, 7} = 209, byte1 = bits {11, 15} = 136, byte2 = bits {19, 21, 22} = 104
    ct = np.array([1, 2, 3, 4, 0, 1, 2, 3, 0, 0, 0, 0, 0, 0, 0, 0], dtype=np.uint64).reshape(1, 2, 1, 8)
    msg = message.pack(ct, [5])
    assert list(msg) == [209, 136, 104, 0, 0, 0]
    assert np.array_equal(message.unpack(msg, 1, 8, [5]), ct)


def test_roundtrip_and_size():
    rng = np.random.default_rng(3)
    q = [97, 193, 65537]
    ct = np.stack([rng.integers(0, p, size=(2, 2, 16)) for p in q], axis=2).astype(np.uint64)
    msg = message.pack(ct, q)
    assert len(msg) == message.message_bytes(2, 16, q) == 2 * 2 * 16 * (7 + 8 + 17) // 8
    assert np.array_equal(message.unpack(msg, 2, 16, q), ct)


def test_saving_vs_words():
    for name in ("c2", "c3", "c4"):
        cfg = inp.CONFIGS[name]
        t = nt.plaintext_modulus(cfg.t_bits, cfg.log2N, cfg.t_fixed)
        q = nt.prime_chain(cfg.q_bits, cfg.log2N, exclude=[t])
        per_ct = message.message_bytes(1, cfg.N, q)
        assert per_ct == 2 * cfg.N * sum(p.bit_length() for p in q) // 8
        assert per_ct < 2 * cfg.L * cfg.N * 8
