"""bench.py's input generation and moduli are oracle-free (only its
cpu_baseline leg may use oracle/); here they are checked against the oracle's
C generator and prime search."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from primes import cfg2_modulus, largest_ntt_primes  # noqa: E402


def test_mt19937_64_rows_match_oracle(oracle):
    seeds = [0, 1, 5489, 20260809, 2**63 + 12345, 2**64 - 1]
    raw = bench.mt19937_64_rows(seeds, 1000)
    for s, row in zip(seeds, raw):
        assert np.array_equal(row, oracle.mt19937_64(s, 1000, 0)), s


def test_make_inputs_and_moduli_match_oracle(oracle):
    moduli = bench.cfg3_moduli()
    assert moduli == largest_ntt_primes(50, bench.N, bench.NLIMBS)
    assert bench.cfg2_modulus() == cfg2_modulus()
    x = bench.make_inputs(moduli[:3], 2, 777).reshape(6, bench.N)
    for r in range(6):
        assert np.array_equal(x[r], oracle.mt19937_64(777 + r, bench.N, moduli[r % 3])), r


def test_shard_inputs_are_slices_of_the_batch():
    """A rank's limb range (make_inputs with limb0/nlimbs) holds exactly the
    words of those limbs in the single-GPU batch, [poly][limb][N] order."""
    moduli = bench.cfg3_moduli()[:6]
    full = bench.make_inputs(moduli, 3, 4242, n=64).reshape(3, 6, 64)
    for limb0, nl in ((0, 2), (2, 3), (5, 1)):
        part = bench.make_inputs(moduli, 3, 4242, n=64, limb0=limb0, nlimbs=nl, total_limbs=6)
        assert np.array_equal(part.reshape(3, nl, 64), full[:, limb0:limb0 + nl]), (limb0, nl)


def test_bench_record_primes_match_reference_rule():
    from primes import smallest_ntt_primes

    for bits, n in ((50, 1024), (50, 16384), (30, 64)):
        assert bench.smallest_ntt_primes(bits, n, 2) == smallest_ntt_primes(bits, n, 2)


def test_both_arms_share_the_config_dict():
    for w in (1, 2, 4, 8):
        c = bench.workload_config(w)
        assert c == bench.workload_config(w) and c["rows"] == 2048


def test_config_moduli_match_survey_appendix_a():
    """bench.py's moduli for cfg1, cfg2, cfg4 and the ends of cfg3."""
    assert bench.largest_ntt_primes(50, 4096, 1) == [1125899906826241]
    assert bench.cfg2_modulus() == 1152921504606846883
    m3 = bench.cfg3_moduli()
    assert (m3[0], m3[15], m3[31]) == (1125899904679937, 1125899893964801, 1125899884036097)
    m4 = bench.largest_ntt_primes(60, 65536, 24)
    assert (m4[0], m4[23]) == (1152921504606584833, 1152921504559267841)
