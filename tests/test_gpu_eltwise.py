"""GPU parity: element-wise kernels and poly multiply against the oracle.

Mirrors tests/test_eltwise.cpp and tests/test_ring.cpp of the reference
(boundary-heavy samplers, float-path correction triples, factor-8 boundary,
FMA known answer, schoolbook and monomial-sign known answers) plus the
BASELINE cfg2 / cfg5 shapes.
"""
import numpy as np
import pytest
import torch

from primes import (cfg2_modulus, cfg5, config_seed, largest_ntt_primes, primes_with_bits,
                    smallest_ntt_primes)

pytestmark = pytest.mark.gpu


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64).view(np.int64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


def sample_inputs(oracle, q, factor, n, seed):
    """Boundary-heavy values in [0, factor*q) (test_eltwise.cpp:22-27)."""
    v = oracle.mt19937_64(seed, n, factor * q)
    edges = [0, 1, q - 1, q % (factor * q), factor * q - 1]
    for i, e in enumerate(edges[:n]):
        v[i] = e
    return v


MULT_QS = [17, 97] + [primes_with_bits(b, 1)[0] for b in (20, 30, 49, 50, 58, 60, 61, 62)]


@pytest.mark.parametrize("q", MULT_QS)
@pytest.mark.parametrize("fin", [1, 2, 4])
@pytest.mark.parametrize("n", [1, 2, 7, 2048, 4097])
def test_mult_matches_oracle(nk, oracle, q, fin, n):
    if fin * q >= (1 << 63):
        with pytest.raises(ValueError, match="input_mod_factor\\*q < 2\\^63"):
            nk.eltwise_mult_mod(torch.empty(n, dtype=torch.int64, device="cuda"),
                                dev(np.zeros(n)), dev(np.zeros(n)), q, fin)
        return
    a = sample_inputs(oracle, q, fin, n, 11 + n)
    b = sample_inputs(oracle, q, fin, n, 12 + n)
    r = torch.empty(n, dtype=torch.int64, device="cuda")
    nk.eltwise_mult_mod(r, dev(a), dev(b), q, fin)
    want = oracle.eltwise_mult_mod(a, b, q, fin)
    assert np.array_equal(host(r), want)
    # int and float reference paths agree where both apply
    if q < (1 << 50):
        assert np.array_equal(want, oracle.eltwise_mult_mod(a, b, q, fin, path=1))


@pytest.mark.parametrize("q", [17, 97] + [primes_with_bits(b, 1)[0] for b in (20, 30, 49, 50)])
@pytest.mark.parametrize("fin", [1, 2, 4])
@pytest.mark.parametrize("n", [1, 5, 4097])
def test_mult_explicit_paths(nk, oracle, q, fin, n):
    """eltwise_mult_mod_int / _float (eltwise.hpp:137-175): both paths give the
    reference's words wherever they apply."""
    a = sample_inputs(oracle, q, fin, n, 31 + n)
    b = sample_inputs(oracle, q, fin, n, 32 + n)
    want = oracle.eltwise_mult_mod(a, b, q, fin)
    for fn in (nk.eltwise_mult_mod_int, nk.eltwise_mult_mod_float):
        if fn is nk.eltwise_mult_mod_float and q >= (1 << 50):
            continue
        r = torch.empty(n, dtype=torch.int64, device="cuda")
        fn(r, dev(a), dev(b), q, fin)
        assert np.array_equal(host(r), want), fn.__name__
        assert np.array_equal(fn(None, a, b, q, fin), want), fn.__name__ + " (host buffers)"


def _prime_near(oracle, x, step):
    c = x | 1
    while not oracle.is_prime(c):
        c += step
    return c


@pytest.mark.parametrize("fin", [1, 2, 4])
def test_mult_loose_barrett_boundary(nk, oracle, fin):
    """The integer multiply takes loose Barrett quotients for 5q < 2^63 and the
    exact ones above: primes on both sides of 2^63 / 5, boundary-heavy inputs."""
    edge = (1 << 63) // 5
    for q in (_prime_near(oracle, edge, -2), _prime_near(oracle, edge + 2, 2)):
        if fin * q >= (1 << 63):
            continue
        n = 4099
        a = sample_inputs(oracle, q, fin, n, 41)
        b = sample_inputs(oracle, q, fin, n, 42)
        r = torch.empty(n, dtype=torch.int64, device="cuda")
        nk.eltwise_mult_mod(r, dev(a), dev(b), q, fin)
        assert np.array_equal(host(r), oracle.eltwise_mult_mod(a, b, q, fin)), hex(q)


def test_float_path_correction_cases(nk, oracle):
    """test_eltwise.cpp:117-133: quotient estimate overshoot triples."""
    cases = [(1125899906842597, 1006683697935267, 1120468225943409),
             (1125899906842201, 549202230126986, 905685617713605),
             (562949953421381, 526777231650305, 71630581939326),
             (1099511627689, 611973561147, 954725405533)]
    for q, x, y in cases:
        got = nk.eltwise_mult_mod(None, np.array([x], np.uint64), np.array([y], np.uint64), q, 1)
        assert int(got[0]) == (x * y) % q


def test_mult_identities(nk, oracle):
    """test_eltwise.cpp:80-93."""
    q = primes_with_bits(50, 1)[0]
    a = oracle.mt19937_64(35, 256, 4 * q)
    ones = np.ones(256, np.uint64)
    got = nk.eltwise_mult_mod(None, a, ones, q, 4)
    assert np.array_equal(got, a % np.uint64(q))
    top = np.full(256, q - 1, np.uint64)
    assert np.all(nk.eltwise_mult_mod(None, top, top, q, 1) == 1)


FMA_QS = [17] + [primes_with_bits(b, 1)[0] for b in (20, 30, 48, 50, 60)] + [(1 << 61) - 1]  # 2^61 - 1: largest allowed q


@pytest.mark.parametrize("q", FMA_QS)
@pytest.mark.parametrize("fin", [1, 2, 4, 8])
@pytest.mark.parametrize("bs", [0, 52, 64])
@pytest.mark.parametrize("with_z", [True, False])
def test_fma_matches_oracle(nk, oracle, q, fin, bs, with_z):
    n = 1027
    width = bs or (52 if fin * q < (1 << 52) else 64)
    a = sample_inputs(oracle, q, fin, n, 45 + fin)
    z = sample_inputs(oracle, q, fin, n, 46 + fin) if with_z else None
    y = int(oracle.mt19937_64(47 + fin, 1, q)[0])
    r = torch.empty(n, dtype=torch.int64, device="cuda")
    if fin * q >= (1 << width):
        with pytest.raises(ValueError, match="BitShift"):
            nk.eltwise_fma_mod(r, dev(a), y, None if z is None else dev(z), q, fin, bs)
        return
    nk.eltwise_fma_mod(r, dev(a), y, None if z is None else dev(z), q, fin, bs)
    want = oracle.eltwise_fma_mod(a, y, z, q, fin, bs)
    assert np.array_equal(host(r), want)
    exact = [(int(x) * y + (0 if z is None else int(zz))) % q
             for x, zz in zip(a[:64], (z if z is not None else np.zeros(64, np.uint64))[:64])]
    assert [int(v) for v in want[:64]] == exact


def test_fma_known_answers(nk):
    """test_eltwise.cpp:180-208: 2*3+4 mod 17 = 10; factor-8 boundary."""
    out = nk.eltwise_fma_mod(None, np.array([2], np.uint64), 3, np.array([4], np.uint64), 17, 1)
    assert int(out[0]) == 10
    for bits in (20, 50, 60):
        q = primes_with_bits(bits, 1)[0]
        a = np.full(4, 8 * q - 1, np.uint64)
        got = nk.eltwise_fma_mod(None, a, q - 1, a, q, 8)
        assert all(int(v) == ((8 * q - 1) * (q - 1) + 8 * q - 1) % q for v in got)


def test_add_neg(nk, oracle):
    q = primes_with_bits(61, 1)[0]
    a = oracle.mt19937_64(31, 4096, q)
    b = oracle.mt19937_64(32, 4096, q)
    r = torch.empty(4096, dtype=torch.int64, device="cuda")
    nk.eltwise_add_mod(r, dev(a), dev(b), q)
    assert np.array_equal(host(r), oracle.eltwise_add_mod(a, b, q))
    a[0] = 0
    nk.eltwise_neg_mod(r, dev(a), q)
    assert np.array_equal(host(r), oracle.eltwise_neg_mod(a, q))


def test_add_neg_host_buffers(nk, oracle):
    """eltwise_add_mod / eltwise_neg_mod through the host-buffer entry points."""
    q = primes_with_bits(60, 1)[0]
    n = 70001
    a = oracle.mt19937_64(61, n, q)
    b = oracle.mt19937_64(62, n, q)
    a[:3] = [0, q - 1, 1]
    b[:3] = [0, q - 1, q - 1]
    assert np.array_equal(nk.eltwise_add_mod(None, a, b, q), oracle.eltwise_add_mod(a, b, q))
    assert np.array_equal(nk.eltwise_neg_mod(None, a, q), oracle.eltwise_neg_mod(a, q))


def test_cfg2_full(nk, oracle):
    """BASELINE cfg2: 2^20 words, q = largest prime < 2^60, fin 1: vector-vector,
    vector-scalar (FMA without addend) and FMA."""
    q = cfg2_modulus()
    assert q == 1152921504606846883
    n = 1 << 20
    s = config_seed(2)
    a = oracle.mt19937_64(s, n, q)
    b = oracle.mt19937_64(s + 1, n, q)
    z = oracle.mt19937_64(s + 2, n, q)
    y = int(oracle.mt19937_64(s + 3, 1, q)[0])
    r = torch.empty(n, dtype=torch.int64, device="cuda")
    nk.eltwise_mult_mod(r, dev(a), dev(b), q, 1)
    assert np.array_equal(host(r), oracle.eltwise_mult_mod(a, b, q, 1))
    nk.eltwise_fma_mod(r, dev(a), y, None, q, 1)
    assert np.array_equal(host(r), oracle.eltwise_fma_mod(a, y, None, q, 1))
    nk.eltwise_fma_mod(r, dev(a), y, dev(z), q, 1)
    assert np.array_equal(host(r), oracle.eltwise_fma_mod(a, y, z, q, 1))


# ---------------------------------------------------------------------------
# ring
# ---------------------------------------------------------------------------
def test_poly_known_answers(nk):
    """test_ring.cpp: X * X^(n-1) = -1, monomial sign table, ring identity."""
    t = nk.NttTables(8, nk.Modulus(97))
    for i in range(8):
        for j in range(8):
            xi = np.zeros(8, np.uint64)
            xj = np.zeros(8, np.uint64)
            xi[i] = 1
            xj[j] = 1
            want = np.zeros(8, np.uint64)
            if i + j < 8:
                want[i + j] = 1
            else:
                want[i + j - 8] = 96
            assert np.array_equal(nk.poly_mult_mod(None, xi, xj, t), want), (i, j)


@pytest.mark.parametrize("logn", [1, 2, 4, 6, 8])
@pytest.mark.parametrize("bits", [20, 30, 50, 61])
def test_poly_matches_naive(nk, oracle, logn, bits):
    """test_ring.cpp:80-98."""
    n = 1 << logn
    q = smallest_ntt_primes(bits, n, 1)[0]
    t = nk.NttTables(n, nk.Modulus(q))
    for rep in range(3):
        f = oracle.mt19937_64(53 + rep, n, q)
        g = oracle.mt19937_64(54 + rep, n, q)
        f[0] = q - 1
        assert np.array_equal(nk.poly_mult_mod(None, f, g, t), oracle.naive_negacyclic(f, g, q))


def test_poly_alias_and_errors(nk, oracle):
    n = 16
    t = nk.NttTables(n, nk.Modulus(97))
    f = oracle.mt19937_64(57, n, 97)
    g = oracle.mt19937_64(58, n, 97)
    df, dg = dev(f), dev(g)
    want = oracle.poly_mult_mod(n, [97], f, g)
    t.poly_mult_mod(df, df, dg)
    assert np.array_equal(host(df), want)
    df = dev(f)
    t.poly_mult_mod(dg, df, dg)  # result aliases g
    assert np.array_equal(host(dg), want)
    q62 = smallest_ntt_primes(62, 16, 1)[0]
    t62 = nk.NttTables(16, nk.Modulus(q62))
    with pytest.raises(ValueError, match="q < 2\\^61"):
        nk.poly_mult_mod(None, f, g, t62)


def test_cfg5_sample(nk, oracle):
    """BASELINE cfg5 layout (N=16384, 16 limbs x 128 pairs): full GPU run, oracle
    on a deterministic sample of 64 row pairs."""
    c = cfg5()
    n, moduli, npolys = c["n"], c["moduli"], c["npolys"]
    plan = nk.RnsNtt(n, moduli)
    L = len(moduli)
    rows = npolys * L
    s = config_seed(5)
    f = np.empty((rows, n), np.uint64)
    g = np.empty((rows, n), np.uint64)
    for r in range(rows):
        f[r] = oracle.mt19937_64(s + 2 * r, n, moduli[r % L])
        g[r] = oracle.mt19937_64(s + 2 * r + 1, n, moduli[r % L])
    df, dg = dev(f.reshape(-1)), dev(g.reshape(-1))
    out = torch.empty_like(df)
    plan.poly_mult_mod(out, df, dg)
    got = host(out).reshape(rows, n)
    sample = list(range(0, rows, rows // 64))[:64]
    for r in sample:
        want = oracle.poly_mult_mod(n, [moduli[r % L]], f[r], g[r])
        assert np.array_equal(got[r], want), r


@pytest.mark.parametrize("path", ["single", "single_grp", "pair3", "reference"])
def test_poly_16384_paths_and_aliasing(nk, oracle, path):
    """N = 16384 with 50-bit limbs: the single on-chip kernel (default: the
    two-stream poly_str14; nk_debug_block_kernel(3): the group-exchange
    poly_mul14; forward g to TMEM, forward f, product, inverse), the three-launch sequence
    (nk_debug_block_kernel(0): forward g, forward f with the dyadic product in
    its store, inverse) and the reference's fwd(1,4)/mult(4)/inv(1,1) sequence
    (exact_only). All must equal the oracle, also when the result aliases f or
    g and for all-(q-1) and all-zero rows."""
    from primes import largest_ntt_primes

    n = 16384
    moduli = largest_ntt_primes(50, n, 3)
    plan = nk.RnsNtt(n, moduli)
    nk.set_exact_only(path == "reference")
    nk.set_block_kernel({"pair3": 0, "single_grp": 3}.get(path, -1))
    try:
        npolys = 2
        rows = npolys * len(moduli)
        f = np.stack([oracle.mt19937_64(70 + r, n, moduli[r % 3]) for r in range(rows)]).reshape(-1)
        g = np.stack([oracle.mt19937_64(170 + r, n, moduli[r % 3]) for r in range(rows)]).reshape(-1)
        g[:n] = moduli[0] - 1  # extreme rows
        f[n:2 * n] = moduli[1] - 1
        g[n:2 * n] = moduli[1] - 1
        f[2 * n:3 * n] = 0
        want = np.concatenate([oracle.poly_mult_mod(n, [moduli[r % 3]], f[r * n:(r + 1) * n],
                                                    g[r * n:(r + 1) * n]) for r in range(rows)])
        df, dg = dev(f), dev(g)
        out = torch.empty_like(df)
        plan.poly_mult_mod(out, df, dg)
        assert np.array_equal(host(out), want)
        plan.poly_mult_mod(df, df, dg)  # result aliases f
        assert np.array_equal(host(df), want)
        df = dev(f)
        plan.poly_mult_mod(dg, df, dg)  # result aliases g
        assert np.array_equal(host(dg), want)
    finally:
        nk.set_exact_only(False)
        nk.set_block_kernel(-1)


@pytest.mark.parametrize("rows_per_limb", [1, 100, 149])
def test_poly_16384_single_kernel_shapes(nk, oracle, rows_per_limb):
    """The single-kernel poly_mult_mod over a limb sub-range (limb0 = 1 of 4
    limbs) with fewer rows than SMs, about one per SM, and more than SMs (CTAs
    looping over rows); one kernel launch per call."""
    from primes import largest_ntt_primes

    n = 16384
    moduli = largest_ntt_primes(50, n, 4)
    plan = nk.RnsNtt(n, moduli)
    sub = moduli[1:3]
    rows = rows_per_limb * len(sub)
    f = np.stack([oracle.mt19937_64(900 + r, n, sub[r % 2]) for r in range(rows)])
    g = np.stack([oracle.mt19937_64(5900 + r, n, sub[r % 2]) for r in range(rows)])
    df, dg = dev(f.reshape(-1)), dev(g.reshape(-1))
    out = torch.empty_like(df)
    before = nk.launch_count()
    plan.poly_mult_mod(out, df, dg, limb0=1, nlimbs=2)
    torch.cuda.synchronize()
    assert nk.launch_count() - before == 1
    got = host(out).reshape(rows, n)
    for r in sorted({0, 1, rows // 2, rows - 2, rows - 1}):
        want = oracle.poly_mult_mod(n, [sub[r % 2]], f[r], g[r])
        assert np.array_equal(got[r], want), r


def test_poly_16384_unaligned_operands_fall_back(nk, oracle):
    """The single kernel loads f and g with TMA (16-byte aligned rows); 8-byte
    aligned views take the multi-launch sequence instead, same result."""
    from primes import largest_ntt_primes

    n = 16384
    moduli = largest_ntt_primes(50, n, 2)
    rows = 4
    f = np.concatenate([oracle.mt19937_64(80 + r, n, moduli[r % 2]) for r in range(rows)])
    g = np.concatenate([oracle.mt19937_64(90 + r, n, moduli[r % 2]) for r in range(rows)])
    want = oracle.poly_mult_mod(n, moduli, f, g)
    plan = nk.RnsNtt(n, moduli)
    words = f.size
    fb = torch.zeros(words + 1, dtype=torch.int64, device="cuda")
    fb[1:] = dev(f)
    out = torch.empty(words, dtype=torch.int64, device="cuda")
    before = nk.launch_count()
    plan.poly_mult_mod(out, fb[1:], dev(g))
    torch.cuda.synchronize()
    assert nk.launch_count() - before > 1
    assert np.array_equal(host(out), want)


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_unaligned_views(nk, oracle, offset):
    """Device views that start at any word (8/16/32-byte alignment): the
    element-wise kernels pick their vector width, the transforms stage through
    an aligned copy; results equal the aligned ones."""
    from primes import cfg2_modulus, largest_ntt_primes

    q = cfg2_modulus()
    n = 4099
    a = oracle.mt19937_64(91, n, q)
    b = oracle.mt19937_64(92, n, q)
    base_a = torch.zeros(n + 8, dtype=torch.int64, device="cuda")
    base_b = torch.zeros(n + 8, dtype=torch.int64, device="cuda")
    base_r = torch.zeros(n + 8, dtype=torch.int64, device="cuda")
    da, db, dr = base_a[offset:offset + n], base_b[offset:offset + n], base_r[offset:offset + n]
    da.copy_(dev(a))
    db.copy_(dev(b))
    nk.eltwise_mult_mod(dr, da, db, q, 1)
    assert np.array_equal(host(dr), oracle.eltwise_mult_mod(a, b, q, 1))
    nk.eltwise_fma_mod(dr, da, 12345, db, q, 1)
    assert np.array_equal(host(dr), oracle.eltwise_fma_mod(a, 12345, b, q, 1))
    nn = 16384
    qq = largest_ntt_primes(50, nn, 1)[0]
    plan = nk.RnsNtt(nn, [qq])
    x = oracle.mt19937_64(93, nn, qq)
    bx = torch.zeros(nn + 8, dtype=torch.int64, device="cuda")
    bo = torch.zeros(nn + 8, dtype=torch.int64, device="cuda")
    dx, do = bx[offset:offset + nn], bo[offset:offset + nn]
    dx.copy_(dev(x))
    plan.forward(do, dx, 1, 1)
    assert np.array_equal(host(do), oracle.forward(nn, [qq], x, 1, 1))


def test_host_pipeline_multi_chunk(nk, oracle):
    """Host-buffer entry points cut large inputs into ~16 MiB chunks that are
    uploaded / computed / downloaded on two streams: results must not depend on
    the chunking (odd chunk counts, a short last chunk)."""
    from primes import cfg2_modulus, largest_ntt_primes

    q = cfg2_modulus()
    n = 5 * (1 << 20) + 12345  # 3 chunks, the last one short
    a = oracle.mt19937_64(301, n, q)
    b = oracle.mt19937_64(302, n, q)
    got = nk.eltwise_mult_mod(None, a, b, q, 1)
    assert np.array_equal(got, oracle.eltwise_mult_mod(a, b, q, 1))
    got = nk.eltwise_fma_mod(None, a, 987654321, b, q, 1)
    assert np.array_equal(got, oracle.eltwise_fma_mod(a, 987654321, b, q, 1))
    nn = 16384
    moduli = largest_ntt_primes(50, nn, 3)
    plan = nk.RnsNtt(nn, moduli)
    npolys = 45  # 135 rows = 17.6 MiB: two chunks
    x = np.concatenate([oracle.mt19937_64(400 + r, nn, moduli[r % 3]) for r in range(3 * npolys)])
    f = plan.forward(None, x, 1, 1)
    assert np.array_equal(f, oracle.forward(nn, moduli, x, 1, 1, threads=8))
    assert np.array_equal(plan.inverse(None, f, 1, 1), x)


def test_host_pipeline_ramped_chunks(nk, oracle):
    """Long host-buffer runs (at least four full chunks) start and end with a
    quarter and a half chunk: results must match, for words and for whole
    polynomials, with an odd remainder in the middle."""
    from primes import cfg2_modulus, largest_ntt_primes

    q = cfg2_modulus()
    n = 9 * (1 << 21) + 4321  # 4.5 full 16 MiB chunks of words
    a = oracle.mt19937_64(311, n, q)
    b = oracle.mt19937_64(312, n, q)
    assert np.array_equal(nk.eltwise_mult_mod(None, a, b, q, 1), oracle.eltwise_mult_mod(a, b, q, 1))
    nn = 16384
    moduli = largest_ntt_primes(50, nn, 8)  # 1 MiB polynomials: 16 per full chunk
    plan = nk.RnsNtt(nn, moduli)
    npolys = 71
    x = np.concatenate([oracle.mt19937_64(500 + r, nn, moduli[r % 8]) for r in range(8 * npolys)])
    f = plan.forward(None, x, 1, 1)
    assert np.array_equal(f, oracle.forward(nn, moduli, x, 1, 1, threads=8))
    assert np.array_equal(plan.inverse(None, f, 1, 1), x)


def test_eltwise_writes_stay_in_bounds(nk, oracle):
    """Guard words around element-wise and poly-multiply results (see
    test_gpu_ntt.test_writes_stay_in_bounds), odd lengths and offsets."""
    sentinel = np.uint64(0x5A5A5A5A5A5A5A5A)
    guard = 1024
    for q in (primes_with_bits(60, 1)[0], primes_with_bits(49, 1)[0]):
        for n in (1, 7, 4097, 70001):
            a, b = oracle.mt19937_64(5, n, q), oracle.mt19937_64(6, n, q)
            for name, run, want in (
                ("mult", lambda o: nk.eltwise_mult_mod(o, dev(a), dev(b), q, 1), oracle.eltwise_mult_mod(a, b, q, 1)),
                ("fma", lambda o: nk.eltwise_fma_mod(o, dev(a), 3, dev(b), q, 1), oracle.eltwise_fma_mod(a, 3, b, q, 1)),
                ("vs", lambda o: nk.eltwise_fma_mod(o, dev(a), 3, None, q, 1), oracle.eltwise_fma_mod(a, 3, None, q, 1)),
                ("add", lambda o: nk.eltwise_add_mod(o, dev(a), dev(b), q), oracle.eltwise_add_mod(a, b, q)),
                ("neg", lambda o: nk.eltwise_neg_mod(o, dev(a), q), oracle.eltwise_neg_mod(a, q)),
            ):
                for off in (0, 1):
                    buf = torch.full((n + 2 * guard + 1,), int(sentinel.view(np.int64)), dtype=torch.int64,
                                     device="cuda")
                    run(buf[guard + off:guard + off + n])
                    h = host(buf)
                    assert np.all(h[:guard + off] == sentinel), (name, n, off)
                    assert np.all(h[guard + off + n:] == sentinel), (name, n, off)
                    assert np.array_equal(h[guard + off:guard + off + n], want), (name, n, off)
    # fused poly multiply (N = 16384) and the sequence path (N = 1024)
    for n in (1024, 16384):
        moduli = largest_ntt_primes(50, n, 2)
        f = np.concatenate([oracle.mt19937_64(50 + r, n, moduli[r % 2]) for r in range(4)])
        g = np.concatenate([oracle.mt19937_64(60 + r, n, moduli[r % 2]) for r in range(4)])
        plan = nk.RnsNtt(n, moduli)
        words = f.size
        buf = torch.full((words + 2 * guard,), int(sentinel.view(np.int64)), dtype=torch.int64, device="cuda")
        plan.poly_mult_mod(buf[guard:guard + words], dev(f), dev(g))
        h = host(buf)
        assert np.all(h[:guard] == sentinel) and np.all(h[guard + words:] == sentinel)
        assert np.array_equal(h[guard:guard + words], oracle.poly_mult_mod(n, moduli, f, g))
