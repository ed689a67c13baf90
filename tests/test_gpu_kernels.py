"""Standalone kernels of the c5 microbench (BASELINE.json configs[4]) vs the oracle (-m gpu):
forward / inverse negacyclic NTT and the pointwise ct x pt MAC on uniform residues."""
import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import core, nt

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_00737_b200 as eph  # noqa: E402


def _dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("force_int", [False, True])
@pytest.mark.parametrize("log2N", [10, 12, 13, 14, 15, 16])
@pytest.mark.parametrize("L,bits", [(1, 30), (3, 60), (5, 60), (9, 48), (16, 30), (16, 60)])
def test_ntt_fwd_inv_bitexact(log2N, L, bits, force_int):
    # default: the FP64 kernels where the plan's bounds allow them (primes < 2^50),
    # else the integer kernels; force_int: integer only (EPHDC_NTT_FORCE_INT)
    q = nt.prime_chain([bits] * L, log2N)
    batch = 3
    x = inp.gen_residues(q, batch, 1 << log2N, seed=log2N * 100 + L)
    plan = eph.NttPlan(q, log2N, force_int=force_int)
    d = _dev(x)
    eph.ntt_fwd(plan, d)
    got = _host(d)
    for j, p in enumerate(q):
        psi = nt.min_primitive_2n_root(p, 1 << log2N)
        want = core.ntt_fwd(x[:, j, :], log2N, p, psi)
        assert np.array_equal(got[:, j, :], want), (j, p)
    eph.ntt_inv(plan, d)
    assert np.array_equal(_host(d), x)


@pytest.mark.parametrize("log2N,L,bits,D", [(12, 3, 60, 5), (13, 5, 44, 64), (14, 9, 48, 33), (12, 16, 60, 300), (12, 2, 61, 130),
                                            (15, 3, 60, 7), (16, 1, 30, 9), (16, 16, 60, 2),
                                            # integer form, D split beyond floor(2^64 / q) pieces: slot rows
                                            (12, 1, 60, 700), (13, 1, 61, 333), (12, 1, 60, 16)])
def test_mac_bitexact(log2N, L, bits, D):
    N = 1 << log2N
    q = nt.prime_chain([bits] * L, log2N)
    ct = inp.gen_residues(q * 2, D, N, seed=7)                 # [D][2L][N] -> view as [D][L][2][N]
    ct = np.stack([ct[:, 2 * j: 2 * j + 2, :] for j in range(L)], axis=1) % np.array(q, dtype=np.uint64)[None, :, None, None]
    pt = inp.gen_residues(q, D, N, seed=8)
    plan = eph.NttPlan(q, log2N)
    out = _host(eph.mac(plan, _dev(ct), _dev(pt)))
    for j, p in enumerate(q):
        for c in range(2):
            acc = np.zeros(N, dtype=object)
            for d in range(D):
                acc = (acc + ct[d, j, c].astype(object) * pt[d, j].astype(object)) % p
            assert np.array_equal(out[j, c], acc.astype(np.uint64)), (j, c)


@pytest.mark.parametrize("log2N", [12, 13, 14, 15, 16])
def test_ntt_c5_sampled_large_batch(log2N):
    """BASELINE.json configs[4]: a larger batch, parity on the first, the last and
    seeded-random polynomials (independent polynomials: the sample is sound)."""
    N = 1 << log2N
    L, bits = (9, 48) if log2N <= 14 else (5, 60)
    q = nt.prime_chain([bits] * L, log2N)
    batch = max(1, (1 << 22) // (N * L))            # ~32 MB of residues
    x = inp.gen_residues(q, batch, N, seed=4242 + log2N)
    plan = eph.NttPlan(q, log2N)
    d = _dev(x)
    eph.ntt_fwd(plan, d)
    got = _host(d)
    rng = np.random.default_rng(log2N)
    picks = sorted({0, batch - 1, *rng.integers(0, batch, 6).tolist()})
    for b in picks:
        for j, p in enumerate(q):
            psi = nt.min_primitive_2n_root(p, N)
            assert np.array_equal(got[b, j], core.ntt_fwd(x[b, j][None, :], log2N, p, psi)[0]), (b, j)
    eph.ntt_inv(plan, d)
    assert np.array_equal(_host(d), x)


@pytest.mark.parametrize("log2N,L,bits,batch", [(12, 16, 48, 300), (13, 16, 30, 97), (13, 5, 49, 1000),
                                                (14, 9, 48, 77), (14, 3, 44, 400), (12, 1, 48, 1)])
def test_ntt_c5_prime_switch(log2N, L, bits, batch):
    """The persistent c5 kernels walk (prime, polynomial) items prime-major: per CTA the
    range crosses prime boundaries (twiddles reloaded) and the TMA ring wraps many times;
    every polynomial is checked against the oracle on a seeded sample."""
    N = 1 << log2N
    q = nt.prime_chain([bits] * L, log2N)
    x = inp.gen_residues(q, batch, N, seed=9000 + log2N + L)
    plan = eph.NttPlan(q, log2N)
    d = _dev(x)
    eph.ntt_fwd(plan, d)
    got = _host(d)
    rng = np.random.default_rng(batch)
    for b in sorted({0, batch - 1, *rng.integers(0, batch, 5).tolist()}):
        for j in sorted({0, L - 1, int(rng.integers(0, L))}):
            psi = nt.min_primitive_2n_root(q[j], N)
            assert np.array_equal(got[b, j], core.ntt_fwd(x[b, j][None, :], log2N, q[j], psi)[0]), (b, j)
    eph.ntt_inv(plan, d)
    assert np.array_equal(_host(d), x)


@pytest.mark.parametrize("log2N,batch", [(13, 1), (13, 2), (13, 3), (13, 7), (13, 301), (14, 1), (14, 2), (14, 5),
                                         (14, 160), (15, 3), (15, 41), (16, 2), (16, 19)])
def test_ntt_c5_two_groups_equal_one_team(log2N, batch):
    """The two-group c5 kernels (alternate polynomials, group barriers, a segment per
    prime, the TMA ring advanced by the group that frees a buffer; on clusters the
    cross-level outputs pushed by st.async onto the partner's mbarrier, buffer reuse
    signalled by remote arrives) = the one-team kernels, bit for bit, both directions
    (EPHDC_NTT_ALT_TEAMS swaps the layouts), at odd batch sizes (a group with no item,
    one-item segments)."""
    N, L = 1 << log2N, 3
    q = nt.prime_chain([48 if log2N <= 14 else 44] * L, log2N)
    x = inp.gen_residues(q, batch, N, seed=77 + batch + log2N)
    p2, p1 = eph.NttPlan(q, log2N), eph.NttPlan(q, log2N, alt_teams=True)
    assert p2.fwd_kernel == p1.fwd_kernel == "c5_f64" and p2.inv_kernel == "c5_f64"
    d2, d1 = _dev(x), _dev(x)
    eph.ntt_fwd(p2, d2)
    eph.ntt_fwd(p1, d1)
    assert torch.equal(d2, d1)
    b = batch - 1
    psi = nt.min_primitive_2n_root(q[L - 1], N)
    assert np.array_equal(_host(d2)[b, L - 1], core.ntt_fwd(x[b, L - 1][None, :], log2N, q[L - 1], psi)[0])
    eph.ntt_inv(p2, d2)
    eph.ntt_inv(p1, d1)
    assert torch.equal(d2, d1)
    assert np.array_equal(_host(d2), x)


def test_ntt_c5_cluster_inverse_stress():
    """The FP64 cluster kernels (DSMEM exchanges, cluster barriers / remote mbarrier
    signals, the TMA ring) under repetition: 60 forward + inverse launches at seeded
    random sizes (N = 2^14..2^16, 1..9 primes, 1..300 polynomials), each round trip
    exact, every fifth through the other warp layout (EPHDC_NTT_ALT_TEAMS: the one-team
    cluster forward) as well."""
    rng = np.random.default_rng(4711)
    plans = {}
    for it in range(60):
        log2N = int(rng.integers(14, 17))
        L = int(rng.integers(1, 10))
        batch = int(rng.integers(1, 301 if log2N == 14 else 81))
        key = (log2N, L)
        if key not in plans:
            q = nt.prime_chain([48 if log2N == 14 else 44] * L, log2N)
            plans[key] = (q, eph.NttPlan(q, log2N), eph.NttPlan(q, log2N, alt_teams=True))
        q, pd, pa = plans[key]
        x = _dev(inp.gen_residues(q, batch, 1 << log2N, seed=it))
        d = x.clone()
        eph.ntt_fwd(pd, d)
        if it % 5 == 0:
            g = d.clone()
            eph.ntt_inv(pa, g)
            assert torch.equal(g, x), (it, log2N, L, batch)
        eph.ntt_inv(pd, d)
        assert torch.equal(d, x), (it, log2N, L, batch)


@pytest.mark.parametrize("log2N", [10, 12, 13, 14, 15, 16])
@pytest.mark.parametrize("L", [1, 5, 16])
def test_ntt_u32_words(log2N, L):
    """30-bit primes on u32 words (ephdc_ntt_fwd32 / inv32 / mac32) bit-exact."""
    N = 1 << log2N
    q = nt.prime_chain([30] * L, log2N)
    x = inp.gen_residues(q, 3, N, seed=log2N + 31 * L)
    plan = eph.NttPlan(q, log2N)
    assert plan.u32_words
    d = torch.from_numpy(x.astype(np.int32)).cuda()
    eph.ntt_fwd32(plan, d)
    got = d.cpu().numpy().astype(np.uint64)
    for j, p in enumerate(q):
        psi = nt.min_primitive_2n_root(p, N)
        assert np.array_equal(got[:, j, :], core.ntt_fwd(x[:, j, :], log2N, p, psi)), j
    eph.ntt_inv32(plan, d)
    assert np.array_equal(d.cpu().numpy().astype(np.uint64), x)
    D = 37
    ct = np.stack([inp.gen_residues(q, D, N, seed=1), inp.gen_residues(q, D, N, seed=2)], axis=2)   # [D][L][2][N]
    pt = inp.gen_residues(q, D, N, seed=3)
    out = eph.mac32(plan, torch.from_numpy(ct.astype(np.int32)).cuda(), torch.from_numpy(pt.astype(np.int32)).cuda())
    out = out.cpu().numpy().astype(np.uint64)
    for j, p in enumerate(q):
        for c in range(2):
            acc = np.zeros(N, dtype=object)
            for dd in range(D):
                acc = (acc + ct[dd, j, c].astype(object) * pt[dd, j].astype(object)) % p
            assert np.array_equal(out[j, c], acc.astype(np.uint64)), (j, c)


def test_u32_words_need_small_primes():
    q = nt.prime_chain([48], 12)
    plan = eph.NttPlan(q, 12)
    assert not plan.u32_words
    with pytest.raises(eph.EphdcError):
        eph.ntt_fwd32(plan, torch.zeros((1, 1, 4096), dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("log2N", [12, 13, 14, 15, 16])
@pytest.mark.parametrize("L,batch", [(1, 1), (3, 2), (5, 7), (16, 3), (2, 149), (3, 301), (1, 1000)])
def test_ntt_c5_u32_kernels(log2N, L, batch):
    """The persistent TMA-fed u32 kernels (ntt32_c5.cu: swizzled in-place passes, TMEM row
    twiddles, TMA store) = the oracle's NTT on sampled polynomials of every prime, = the
    general u32 kernels (EPHDC_NTT_U32_GENERIC) on the whole batch, and inverse(forward(x))
    = x -- at batches that give CTAs one item, items of two primes, and many items."""
    N = 1 << log2N
    q = nt.prime_chain([30] * L, log2N)
    x = inp.gen_residues(q, batch, N, seed=4000 + 10 * log2N + L + batch)
    pc, pg = eph.NttPlan(q, log2N), eph.NttPlan(q, log2N, u32_generic=True)
    assert pc.u32_kernel == "c5_u32" and pg.u32_kernel == "int_u32"
    dc = torch.from_numpy(x.astype(np.int32)).cuda()
    dg = dc.clone()
    eph.ntt_fwd32(pc, dc)
    eph.ntt_fwd32(pg, dg)
    assert torch.equal(dc, dg)
    got = dc.cpu().numpy().astype(np.uint32).astype(np.uint64)
    rng = np.random.default_rng(batch)
    for b in sorted({0, batch - 1, int(rng.integers(0, batch))}):
        for j in range(L):
            psi = nt.min_primitive_2n_root(q[j], N)
            assert np.array_equal(got[b, j], core.ntt_fwd(x[b, j][None, :], log2N, q[j], psi)[0]), (b, j)
    eph.ntt_inv32(pc, dc)
    eph.ntt_inv32(pg, dg)
    assert torch.equal(dc, dg)
    assert np.array_equal(dc.cpu().numpy().astype(np.uint32).astype(np.uint64), x)


def test_ntt_c5_u32_inverse_vs_oracle():
    """Inverse alone (not only as the forward's inverse) against the oracle's INTT."""
    log2N, L, N = 13, 3, 1 << 13
    q = nt.prime_chain([30] * L, log2N)
    x = inp.gen_residues(q, 5, N, seed=4242)
    p = eph.NttPlan(q, log2N)
    d = torch.from_numpy(x.astype(np.int32)).cuda()
    eph.ntt_inv32(p, d)
    got = d.cpu().numpy().astype(np.uint32).astype(np.uint64)
    for j in range(L):
        psi = nt.min_primitive_2n_root(q[j], N)
        assert np.array_equal(got[:, j], core.ntt_inv(x[:, j], log2N, q[j], psi)), j


def test_ntt_c5_u32_stress_repeated_launches():
    """The TMA/mbarrier ring of ntt32_c5.cu under repetition: 120 forward + inverse
    launches at seeded random sizes (N = 2^12..2^14, 1..16 primes, 1..2500 polynomials),
    each checked to round-trip exactly, every tenth against the general u32 kernels."""
    rng = np.random.default_rng(2024)
    plans = {}
    for it in range(120):
        log2N = int(rng.integers(12, 15))
        L = int(rng.integers(1, 17))
        batch = int(rng.integers(1, 2501 if log2N < 14 else 801))
        key = (log2N, L)
        if key not in plans:
            q = nt.prime_chain([30] * L, log2N)
            plans[key] = (q, eph.NttPlan(q, log2N), eph.NttPlan(q, log2N, u32_generic=True))
        q, pc, pg = plans[key]
        qt = torch.tensor(q, dtype=torch.int64, device="cuda").view(1, L, 1)
        x = torch.remainder(torch.randint(0, 1 << 31, (batch, L, 1 << log2N), device="cuda", dtype=torch.int64), qt)
        x = x.to(torch.int32)
        d = x.clone()
        eph.ntt_fwd32(pc, d)
        if it % 10 == 0:
            g = x.clone()
            eph.ntt_fwd32(pg, g)
            assert torch.equal(d, g), (it, log2N, L, batch)
        eph.ntt_inv32(pc, d)
        assert torch.equal(d, x), (it, log2N, L, batch)


@pytest.mark.parametrize("log2N", [12, 13, 14])
@pytest.mark.parametrize("L,batch", [(1, 1), (3, 7), (16, 3), (2, 301)])
def test_ntt_u64_words_30bit_on_u32_kernels(log2N, L, batch):
    """u64 words with every prime < 2^30 run the u32 kernels on the low words (TMA with
    element stride 2): = the FP64 c5 kernels (EPHDC_NTT_U32_GENERIC keeps those) bit for
    bit, = the oracle on sampled polynomials, high words stay zero, inverse round-trips."""
    N = 1 << log2N
    q = nt.prime_chain([30] * L, log2N)
    x = inp.gen_residues(q, batch, N, seed=5000 + 7 * log2N + L + batch)
    pa, pb = eph.NttPlan(q, log2N), eph.NttPlan(q, log2N, u32_generic=True)
    assert pa.fwd_kernel == pa.inv_kernel == "c5_u32" and pb.fwd_kernel == "c5_f64"
    da, db = _dev(x), _dev(x)
    eph.ntt_fwd(pa, da)
    eph.ntt_fwd(pb, db)
    assert torch.equal(da, db)
    got = _host(da)
    assert int(got.max()) < (1 << 30)
    for b in sorted({0, batch - 1}):
        for j in range(L):
            psi = nt.min_primitive_2n_root(q[j], N)
            assert np.array_equal(got[b, j], core.ntt_fwd(x[b, j][None, :], log2N, q[j], psi)[0]), (b, j)
    eph.ntt_inv(pa, da)
    eph.ntt_inv(pb, db)
    assert torch.equal(da, db)
    assert np.array_equal(_host(da), x)
