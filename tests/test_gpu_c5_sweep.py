"""c5 microbench parity at EVERY point tools/bench_c5.py measures (-m gpu, slow).

BASELINE.json configs[4]: standalone negacyclic NTT forward / inverse and the ct x pt
MAC on uniform residues, N = 2^12 ... 2^16, L in {1, 3, 5, 9, 16}, word classes
(30-bit primes in u64 and in u32 words, 48-bit, 60-bit), batches 1 ... 65536 capped at
the 32 GB working set (ephdc_inputs.c5_points -- the same list and the same seeded
device generator the bench uses).  Per point and batch:
  * forward: the first, the last and seeded-random polynomials bit-exact against the
    oracle's NTT (independent polynomials: the sample is sound);
  * inverse(forward(x)) == x for EVERY polynomial of the batch;
  * MAC: seeded coefficient positions of every (prime, component) equal the sum of
    products mod q written out with Python integers over all D terms.
"""
import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import core, nt

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_00737_b200 as eph  # noqa: E402

POINTS = inp.c5_points("all")


def _ids(p):
    lg, L, bits, wb, _ = p
    return f"N{1 << lg}-L{L}-{bits}b-u{8 * wb}"


def _fns(wb):
    return (eph.ntt_fwd, eph.ntt_inv, eph.mac) if wb == 8 else (eph.ntt_fwd32, eph.ntt_inv32, eph.mac32)


@pytest.mark.parametrize("point", POINTS, ids=_ids)
def test_c5_point(point):
    lg, L, bits, wb, batches = point
    N = 1 << lg
    q = nt.prime_chain([bits] * L, lg)
    plan = eph.NttPlan(q, lg)
    fwd, inv, mac = _fns(wb)
    dt = torch.int64 if wb == 8 else torch.int32
    seed = lg * 1000 + L * 10 + bits + wb
    base = inp.c5_residues_torch(q, max(batches), N, seed, "cuda", dt)
    ref = base.clone()
    rng = np.random.default_rng(seed)
    psis = [nt.min_primitive_2n_root(p, N) for p in q]
    for batch in batches:
        x = base[:batch]
        fwd(plan, x)
        for b in sorted({0, batch - 1, *rng.integers(0, batch, 3).tolist()}):
            got = x[b].cpu().numpy().astype(np.uint64) & np.uint64((1 << (8 * wb)) - 1)
            src = ref[b].cpu().numpy().astype(np.uint64) & np.uint64((1 << (8 * wb)) - 1)
            for j in sorted({0, L - 1, int(rng.integers(0, L))}):
                want = core.ntt_fwd(src[j][None, :], lg, q[j], psis[j])[0]
                assert np.array_equal(got[j], want), (batch, b, j)
        inv(plan, x)
        assert torch.equal(x, ref[:batch]), batch
    del base, ref
    torch.cuda.empty_cache()
    # MAC over D terms (the bench's D), sampled positions checked with Python integers
    cap = inp.c5_max_batch(lg, L, wb)
    D = max(1, min(cap, (2 << 30) // (3 * L * N * wb)))
    # ct [D][L][2][N]: rows (j, c) uniform below q_j
    mods = [q[j] for j in range(L) for _ in range(2)]
    ct = inp.c5_residues_torch(mods, D, N, seed + 1, "cuda", dt).view(D, L, 2, N)
    pt = inp.c5_residues_torch(q, D, N, seed + 2, "cuda", dt)
    out = mac(plan, ct, pt)
    outh = out.cpu().numpy().astype(np.uint64) & np.uint64((1 << (8 * wb)) - 1)
    pos = rng.integers(0, N, 4)
    cth = ct[:, :, :, pos].cpu().numpy().astype(object) & ((1 << (8 * wb)) - 1)
    pth = pt[:, :, pos].cpu().numpy().astype(object) & ((1 << (8 * wb)) - 1)
    for j in range(L):
        for c in range(2):
            want = [int(sum(int(a) * int(b) for a, b in zip(cth[:, j, c, t], pth[:, j, t])) % q[j]) for t in range(4)]
            assert [int(v) for v in outh[j, c, pos]] == want, (j, c)
