"""GPU parity: the sm_100a NTT kernels (through the C-ABI) against the CPU
oracle, bit for bit, canonical AND lazy outputs.

Mirrors the reference's tests/test_ntt.cpp cases (known answers, lifted inputs
across (fin, fout), round trips, accumulator widths, maximum size) and adds the
batched RNS shapes of the BASELINE configs.
"""
import numpy as np
import pytest
import torch

from primes import largest_ntt_primes, smallest_ntt_primes, config_seed, cfg3, cfg4

pytestmark = pytest.mark.gpu

FWD_FACTORS = [(1, 1), (1, 4), (2, 1), (2, 4), (4, 1), (4, 4)]
INV_FACTORS = [(1, 1), (1, 2), (2, 1), (2, 2)]


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


def lifted(oracle, x, moduli, n, fin, seed):
    """x + q*r with r < fin, per row modulus (test_ntt.cpp:164-166)."""
    if fin == 1:
        return x.copy()
    r = oracle.mt19937_64(seed, x.size, fin)
    q = np.repeat(np.asarray(moduli, dtype=np.uint64), n)
    q = np.tile(q, x.size // q.size)
    return x + q * r


def rows_of(oracle, moduli, n, npolys, seed):
    """[npolys][nlimbs][n], row limb l uniform in [0, q_l)."""
    out = np.empty((npolys, len(moduli), n), np.uint64)
    k = 0
    for p in range(npolys):
        for l, q in enumerate(moduli):
            out[p, l] = oracle.mt19937_64(seed + 1000 * k, n, q)
            k += 1
    return out.reshape(-1)


def check_dir(nk, oracle, n, moduli, npolys, seed, fwd_factors=FWD_FACTORS,
              inv_factors=INV_FACTORS, bit_shift=0):
    plan = nk.RnsNtt(n, moduli, bit_shift=bit_shift)
    x = rows_of(oracle, moduli, n, npolys, seed)
    for fin, fout in fwd_factors:
        xi = lifted(oracle, x, moduli, n, fin, seed + fin)
        d = dev(xi)
        out = torch.empty_like(d)
        plan.forward(out, d, fin, fout)
        want = oracle.forward(n, moduli, xi, fin, fout, bit_shift=bit_shift, threads=8)
        got = host(out)
        assert np.array_equal(got, want), f"fwd n={n} fin={fin} fout={fout} mism={np.sum(got != want)}"
        # in place
        plan.forward(d, d, fin, fout)
        assert np.array_equal(host(d), want)
    for fin, fout in inv_factors:
        xi = lifted(oracle, x, moduli, n, fin, seed + 7 * fin)
        d = dev(xi)
        out = torch.empty_like(d)
        plan.inverse(out, d, fin, fout)
        want = oracle.inverse(n, moduli, xi, fin, fout, bit_shift=bit_shift, threads=8)
        got = host(out)
        assert np.array_equal(got, want), f"inv n={n} fin={fin} fout={fout} mism={np.sum(got != want)}"


@pytest.mark.parametrize("logn", list(range(1, 11)))
@pytest.mark.parametrize("bits", [20, 30, 50, 61])
def test_small_sizes_match_oracle(nk, oracle, logn, bits, arith):
    n = 1 << logn
    moduli = smallest_ntt_primes(bits, n, 2)
    check_dir(nk, oracle, n, moduli, 3, 100 + logn * 7 + bits)


@pytest.fixture(params=[False, True], ids=["auto", "exact_only"])
def arith(request, nk):
    """Canonical-output beta = 2^52 transforms run signed FP64 arithmetic by
    default; exact_only forces the lazy-exact arithmetic on them too."""
    nk.set_exact_only(request.param)
    yield request.param
    nk.set_exact_only(False)


@pytest.mark.parametrize("logn", [11, 12, 13, 14])
@pytest.mark.parametrize("bits", [30, 50, 60, 61])
def test_block_sizes_match_oracle(nk, oracle, logn, bits, arith):
    n = 1 << logn
    moduli = largest_ntt_primes(bits, n, 3)
    check_dir(nk, oracle, n, moduli, 2, 300 + logn * 7 + bits)


@pytest.mark.parametrize("logn", [1, 3, 10, 12, 14])
@pytest.mark.parametrize("pattern", ["max", "zero", "alt", "top"])
def test_extreme_inputs(nk, oracle, logn, pattern, arith):
    """Worst-case magnitudes for the lazy/signed bounds: all q-1 (lifted to
    fin*q - 1), zeros, alternating 0 / max, and max in the top half only."""
    n = 1 << logn
    moduli = largest_ntt_primes(50, n, 2)
    plan = nk.RnsNtt(n, moduli)
    q = np.repeat(np.asarray(moduli, dtype=np.uint64), n)
    for fin, fout in FWD_FACTORS + [(f, o) for f, o in INV_FACTORS]:
        top = q * np.uint64(fin) - np.uint64(1)
        if pattern == "max":
            x = top
        elif pattern == "zero":
            x = np.zeros_like(q)
        elif pattern == "alt":
            x = np.where(np.arange(q.size) % 2 == 0, top, np.uint64(0)).astype(np.uint64)
        else:
            x = np.where((np.arange(q.size) % n) >= n // 2, top, np.uint64(0)).astype(np.uint64)
        d = dev(x)
        if (fin, fout) in FWD_FACTORS:
            got = host(plan.forward(torch.empty_like(d), d, fin, fout))
            want = oracle.forward(n, moduli, x, fin, fout)
            assert np.array_equal(got, want), f"fwd {pattern} fin={fin} fout={fout}"
        if (fin, fout) in INV_FACTORS:
            got = host(plan.inverse(torch.empty_like(d), d, fin, fout))
            want = oracle.inverse(n, moduli, x, fin, fout)
            assert np.array_equal(got, want), f"inv {pattern} fin={fin} fout={fout}"


@pytest.mark.parametrize("logn", [15, 16, 17, 18])
@pytest.mark.parametrize("bits", [50, 60])
def test_long_rows_match_oracle(nk, oracle, logn, bits):
    n = 1 << logn
    moduli = largest_ntt_primes(bits, n, 2)
    check_dir(nk, oracle, n, moduli, 1, 500 + logn + bits,
              fwd_factors=[(1, 1), (1, 4), (4, 1), (2, 4)], inv_factors=[(1, 1), (2, 1), (1, 2)])


def test_maximum_size_round_trip(nk, oracle):
    """test_ntt.cpp:335-347: N = 2^20 forward then inverse is the identity; plus
    one direction against the oracle."""
    n = 1 << 20
    q = smallest_ntt_primes(50, n, 1)[0]
    plan = nk.RnsNtt(n, [q])
    x = oracle.mt19937_64(21, n, q)
    d = dev(x)
    f = plan.forward(torch.empty_like(d), d, 1, 1)
    assert np.array_equal(host(f), oracle.forward(n, [q], x, 1, 1))
    b = plan.inverse(torch.empty_like(d), f, 1, 1)
    assert np.array_equal(host(b), x)


@pytest.mark.parametrize("n", [64, 4096, 16384])
def test_accumulator_widths(nk, oracle, n):
    """Forced beta = 2^64 tables on a 50-bit prime agree with the oracle using the
    same width; canonical outputs agree across widths (test_ntt.cpp:228-248)."""
    moduli = largest_ntt_primes(49, n, 2)
    check_dir(nk, oracle, n, moduli, 2, 77, bit_shift=64)
    check_dir(nk, oracle, n, moduli, 2, 78, bit_shift=52)


def test_mixed_width_limbs(nk, oracle):
    """One plan with 50-bit (beta 2^52) and 60-bit (beta 2^64) limbs."""
    n = 4096
    moduli = [largest_ntt_primes(50, n, 1)[0], largest_ntt_primes(60, n, 1)[0],
              largest_ntt_primes(40, n, 1)[0]]
    check_dir(nk, oracle, n, moduli, 3, 91)


def test_known_answers(nk):
    """test_ntt.cpp:80-114: zero, delta and the n=2, q=5 by-hand vectors."""
    t = nk.NttTables(2, nk.Modulus(5))
    assert t.root() == 2
    assert list(t.forward(None, np.array([1, 1], np.uint64), 1, 1)) == [3, 4]
    assert list(t.inverse(None, np.array([3, 4], np.uint64), 1, 1)) == [1, 1]
    assert list(t.inverse(None, np.zeros(2, np.uint64), 1, 1)) == [0, 0]
    t8 = nk.NttTables(8, nk.Modulus(97))
    assert list(t8.forward(None, np.zeros(8, np.uint64), 1, 1)) == [0] * 8
    delta = np.zeros(8, np.uint64)
    delta[0] = 42
    assert list(t8.forward(None, delta, 1, 1)) == [42] * 8


def test_custom_root(nk, oracle):
    """NttTables(n, m, root) with a non-minimal primitive root (ntt.hpp:212-213)."""
    n = 1024
    q = largest_ntt_primes(50, n, 1)[0]
    psi = oracle.minimal_primitive_root(2 * n, q)
    root = oracle.lib.oc_pow_mod(psi, 3, q)  # odd power: still primitive
    t = nk.NttTables(n, nk.Modulus(q), root)
    assert t.root() == root
    x = oracle.mt19937_64(3, n, q)
    got = t.forward(None, x, 1, 4)
    assert np.array_equal(got, oracle.forward(n, [q], x, 1, 4, root=root))
    got = t.forward(None, x, 1, 1)
    ref = oracle.reference_ntt(q, root, x, "forward")
    assert np.array_equal(got, ref)


def test_definitional_transform(nk, oracle):
    """Against the O(N^2) definition (ntt.hpp:457-508) at cfg1 size."""
    n = 4096
    q = largest_ntt_primes(50, n, 1)[0]
    t = nk.NttTables(n, nk.Modulus(q))
    x = oracle.mt19937_64(config_seed(1), n, q)
    f = t.forward(None, x, 1, 1)
    assert np.array_equal(f, oracle.reference_ntt(q, t.root(), x, "forward"))
    assert np.array_equal(t.inverse(None, f, 1, 1), x)


def test_cfg3_full(nk, oracle, arith):
    """BASELINE cfg3: N=16384, 32 limbs x 64 polys, forward(1,1) and inverse(1,1)."""
    c = cfg3()
    n, moduli, npolys = c["n"], c["moduli"], c["npolys"]
    plan = nk.RnsNtt(n, moduli)
    x = rows_of(oracle, moduli, n, npolys, config_seed(3))
    d = dev(x)
    f = plan.forward(torch.empty_like(d), d, 1, 1)
    fh = host(f)
    assert np.array_equal(fh, oracle.forward(n, moduli, x, 1, 1, threads=16))
    b = plan.inverse(torch.empty_like(d), f, 1, 1)
    assert np.array_equal(host(b), x)


def test_cfg4_full(nk, oracle):
    """BASELINE cfg4: N=65536, 24 60-bit limbs x 16 polys, fwd(4,1) and inv(2,1)."""
    c = cfg4()
    n, moduli, npolys = c["n"], c["moduli"], c["npolys"]
    plan = nk.RnsNtt(n, moduli)
    x = rows_of(oracle, moduli, n, npolys, config_seed(4))
    x4 = lifted(oracle, x, moduli, n, 4, 44)
    d = dev(x4)
    f = plan.forward(torch.empty_like(d), d, 4, 1)
    fh = host(f)
    assert np.array_equal(fh, oracle.forward(n, moduli, x4, 4, 1, threads=16))
    x2 = lifted(oracle, fh, moduli, n, 2, 45)
    b = plan.inverse(torch.empty_like(d), dev(x2), 2, 1)
    assert np.array_equal(host(b), x)


@pytest.mark.parametrize("kernel", [0, 1, 2], ids=["pair", "grp", "str"])
@pytest.mark.parametrize("logn,bits,npolys", [(14, 50, 3), (14, 60, 2), (15, 50, 1), (16, 60, 1)])
def test_block_kernels_match_oracle(nk, oracle, kernel, logn, bits, npolys, arith):
    """The three 16384-word block kernel families (CTA pair / group exchange /
    two streams per thread, the default), both arithmetic paths, whole rows
    and the low 14 bits of long rows, odd block counts."""
    nk.set_block_kernel(kernel)
    try:
        n = 1 << logn
        moduli = largest_ntt_primes(bits, n, 3)
        check_dir(nk, oracle, n, moduli, npolys, 900 + logn + bits + kernel)
    finally:
        nk.set_block_kernel(-1)


@pytest.mark.parametrize("logn", [10, 11, 12, 13])
@pytest.mark.parametrize("bits", [50, 60])
def test_block_sizes_large_batches(nk, oracle, logn, bits, arith):
    """Batches of >= #SMs rows take the block kernels with 16 or 32 words per
    thread (dispatch.cuh block_logv: chosen per size, policy and direction;
    small batches take the 8-words-per-thread ones,
    test_block_sizes_match_oracle). Canonical and lazy factors, so every
    arithmetic policy runs in both shapes."""
    n = 1 << logn
    moduli = largest_ntt_primes(bits, n, 3)
    check_dir(nk, oracle, n, moduli, 52, 700 + logn, fwd_factors=[(1, 1), (4, 4), (2, 1)],
              inv_factors=[(1, 1), (2, 2)])


@pytest.mark.parametrize("logn", [12, 14, 15, 16])
def test_loose_quotient_boundary(nk, oracle, logn):
    """Canonical beta = 2^64 transforms take the loose-quotient policy
    (ArithIntL) for q < 2^61 and the exact one above: a plan holding the
    largest 61-bit and the smallest 62-bit NTT primes runs both, limb by limb,
    plus single-width plans of each."""
    n = 1 << logn
    q61 = largest_ntt_primes(61, n, 1)
    q62 = smallest_ntt_primes(62, n, 1)
    for moduli in (q61 + q62, q61, q62):
        check_dir(nk, oracle, n, moduli, 1, 900 + logn,
                  fwd_factors=[(1, 1), (4, 1)], inv_factors=[(1, 1), (2, 1)])


def test_shared_tables_across_threads(nk, oracle):
    """test_ntt.cpp:349-375: four threads transform through one shared plan,
    50 times each; here both through the blocking host-buffer calls and
    through device buffers on per-thread streams."""
    import threading

    n = 1024
    q = smallest_ntt_primes(50, n, 1)[0]
    plan = nk.RnsNtt(n, [q])
    k = 4
    inputs = [oracle.mt19937_64(1500 + i, n, q) for i in range(k)]
    expected = [oracle.forward(n, [q], x, 1, 1) for x in inputs]
    host_out = [np.zeros(n, np.uint64) for _ in range(k)]
    dev_out = [None] * k
    errors = []

    def work(i):
        try:
            for _ in range(50):
                plan.forward(host_out[i], inputs[i], 1, 1)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                d = dev(inputs[i])
                o = torch.empty_like(d)
                for _ in range(50):
                    plan.forward(o, d, 1, 1)
                st.synchronize()
                dev_out[i] = o.cpu().numpy().view(np.uint64)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(k)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i in range(k):
        assert np.array_equal(host_out[i], expected[i])
        assert np.array_equal(dev_out[i], expected[i])


@pytest.mark.parametrize("logn", [10, 11, 12, 13])
@pytest.mark.parametrize("bits", [50, 60])
def test_small_batch_plain_block_kernel(nk, oracle, logn, bits):
    """Small batches of 2^11..2^13-word rows normally take the latency kernel
    (ntt_block_lat: staged twiddles, programmatic dependent launch); mode 6
    forces the plain block kernel, which must agree as well."""
    n = 1 << logn
    moduli = largest_ntt_primes(bits, n, 2)
    nk.set_block_kernel(6)
    try:
        check_dir(nk, oracle, n, moduli, 1, 950 + logn + bits)
    finally:
        nk.set_block_kernel(-1)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_limb_shards_on_one_gpu(nk, oracle, world):
    """the multi-GPU partition simulated on one GPU. Each rank's
    contiguous limb range (sharding.limb_shard) of a cfg3-shaped batch
    (N = 16384, 8 limbs, 3 polys) is transformed by its own plan over its
    limbs, as a rank would; the concatenated shards equal the whole-batch
    transform (forward and inverse), and the same holds through the limb0/nlimbs
    sub-range of one full plan."""
    from paper_2103_16400_b200.sharding import limb_shard, shard_rows

    n, nlimbs, npolys = 16384, 8, 3
    moduli = largest_ntt_primes(50, n, nlimbs)
    x = rows_of(oracle, moduli, n, npolys, 4242)
    full_plan = nk.RnsNtt(n, moduli)
    d = dev(x)
    want_f = host(full_plan.forward(torch.empty_like(d), d, 1, 1))
    want_i = host(full_plan.inverse(torch.empty_like(d), d, 1, 1))
    got_f = np.empty((npolys, nlimbs, n), np.uint64)
    got_i = np.empty((npolys, nlimbs, n), np.uint64)
    for rank in range(world):
        l0, cnt = limb_shard(nlimbs, world, rank)
        if cnt == 0:
            continue
        plan = nk.RnsNtt(n, moduli[l0:l0 + cnt])
        xs = dev(shard_rows(x, n, nlimbs, l0, cnt))
        got_f[:, l0:l0 + cnt, :] = host(plan.forward(torch.empty_like(xs), xs, 1, 1)).reshape(npolys, cnt, n)
        got_i[:, l0:l0 + cnt, :] = host(plan.inverse(torch.empty_like(xs), xs, 1, 1)).reshape(npolys, cnt, n)
        # the same shard through the full plan's limb sub-range
        sub = host(full_plan.forward(torch.empty_like(xs), xs, 1, 1, limb0=l0, nlimbs=cnt))
        assert np.array_equal(sub.reshape(npolys, cnt, n), got_f[:, l0:l0 + cnt, :])
    assert np.array_equal(got_f.reshape(-1), want_f)
    assert np.array_equal(got_i.reshape(-1), want_i)
    assert np.array_equal(want_f, oracle.forward(n, moduli, x, 1, 1, threads=8))


SENTINEL = 0x5A5A5A5A5A5A5A5A


@pytest.mark.parametrize("logn,bits,npolys", [(4, 30, 3), (10, 50, 2), (12, 50, 1), (13, 60, 200),
                                              (14, 50, 3), (14, 60, 2), (15, 50, 1), (16, 60, 1)])
def test_writes_stay_in_bounds(nk, oracle, logn, bits, npolys):
    """compute-sanitizer is closed on this GPU pool, so out-of-bounds global
    writes are caught with guard words instead: the result is a view into a
    larger buffer whose words before and after it hold a sentinel, for every
    kernel family (small, block, latency, pair, single-CTA, global pass) and
    both directions, in place and out of place; results still match the
    oracle."""
    n = 1 << logn
    moduli = largest_ntt_primes(bits, n, 2)
    x = rows_of(oracle, moduli, n, npolys, 777 + logn)
    words, guard = x.size, 4096
    plan = nk.RnsNtt(n, moduli)
    for fwd in (True, False):
        buf = torch.full((words + 2 * guard,), SENTINEL, dtype=torch.int64, device="cuda")
        out = buf[guard:guard + words]
        d = dev(x)
        (plan.forward if fwd else plan.inverse)(out, d, 1, 1)
        h = host(buf)
        assert np.all(h[:guard] == np.uint64(SENTINEL)) and np.all(h[guard + words:] == np.uint64(SENTINEL))
        want = (oracle.forward if fwd else oracle.inverse)(n, moduli, x, 1, 1, threads=8)
        assert np.array_equal(h[guard:guard + words], want)
        # in place inside the guarded buffer
        buf = torch.full((words + 2 * guard,), SENTINEL, dtype=torch.int64, device="cuda")
        buf[guard:guard + words] = dev(x)
        mid = buf[guard:guard + words]
        (plan.forward if fwd else plan.inverse)(mid, mid, 1, 1)
        h = host(buf)
        assert np.all(h[:guard] == np.uint64(SENTINEL)) and np.all(h[guard + words:] == np.uint64(SENTINEL))
        assert np.array_equal(h[guard:guard + words], want)


@pytest.mark.parametrize("pinned", [False, True], ids=["pageable", "pinned"])
def test_host_pipeline_multi_chunk_in_place(nk, oracle, pinned):
    """Host-buffer transforms spanning several 16 MiB pipeline chunks, result
    aliasing the operand (ntt.hpp:267-268), from pageable numpy memory (pinned
    staging + parallel host copies) and from pinned memory (direct DMA)."""
    n = 16384
    moduli = largest_ntt_primes(50, n, 3)
    npolys = 100  # 300 rows = 37.5 MiB: three chunks
    plan = nk.RnsNtt(n, moduli)
    x = rows_of(oracle, moduli, n, npolys, 4242)
    want = host(plan.forward(torch.empty_like(dev(x)), dev(x), 1, 1))
    if pinned:
        buf = torch.from_numpy(x.view(np.int64)).pin_memory().numpy().view(np.uint64)
    else:
        buf = x.copy()
    plan.forward(buf, buf, 1, 1)
    assert np.array_equal(buf, want)
    plan.inverse(buf, buf, 1, 1)
    assert np.array_equal(buf, x)
    # element-wise host calls through the same pipeline (two staged inputs)
    q = moduli[0]
    a, b = x[:2_400_000] % np.uint64(q), x[2_400_000:4_800_000] % np.uint64(q)  # two chunks each
    r = nk.eltwise_mult_mod(None, a, b, q, 1)
    assert np.array_equal(r, oracle.eltwise_mult_mod(a, b, q, 1))


@pytest.mark.parametrize("pattern", ["max", "alt", "random"])
def test_signed_policy_bounds_across_moduli(nk, oracle, pattern):
    """The signed FP64 policy's reduced schedules (balanced twiddles, a
    reduction on every other forward stage, none for sums of two products in the
    inverse, modmath.cuh) at the ends of their modulus range: the smallest and
    the largest 50-bit limb, and 40-, 30- and 20-bit limbs, N = 16384, on
    worst-case and random operands, canonical outputs of every input factor,
    and poly_mult_mod of the same operands."""
    n = 1 << 14
    moduli = [smallest_ntt_primes(50, n, 1)[0], largest_ntt_primes(50, n, 1)[0], largest_ntt_primes(40, n, 1)[0],
              largest_ntt_primes(30, n, 1)[0], largest_ntt_primes(20, n, 1)[0]]
    plan = nk.RnsNtt(n, moduli)
    q = np.repeat(np.asarray(moduli, dtype=np.uint64), n)
    base = rows_of(oracle, moduli, n, 1, 77)
    for fin, fout, fwd in [(1, 1, True), (2, 1, True), (4, 1, True), (1, 1, False), (2, 1, False)]:
        top = q * np.uint64(fin) - np.uint64(1)
        if pattern == "max":
            x = top
        elif pattern == "alt":
            x = np.where(np.arange(q.size) % 2 == 0, top, np.uint64(0)).astype(np.uint64)
        else:
            x = lifted(oracle, base, moduli, n, fin, 5 + fin)
        d = dev(x)
        if fwd:
            got = host(plan.forward(torch.empty_like(d), d, fin, fout))
            want = oracle.forward(n, moduli, x, fin, fout)
        else:
            got = host(plan.inverse(torch.empty_like(d), d, fin, fout))
            want = oracle.inverse(n, moduli, x, fin, fout)
        assert np.array_equal(got, want), f"{'fwd' if fwd else 'inv'} {pattern} fin={fin}"
    f = (q - np.uint64(1)) if pattern != "random" else base
    g = f if pattern == "max" else rows_of(oracle, moduli, n, 1, 78)
    df, dg = dev(f), dev(g)
    got = host(plan.poly_mult_mod(torch.empty_like(df), df, dg))
    want = oracle.poly_mult_mod(n, moduli, f, g)
    assert np.array_equal(got, want), f"poly {pattern}"
