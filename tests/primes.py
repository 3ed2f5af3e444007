"""Modulus choice for the BASELINE configs and the reference's test classes.

- ``largest_ntt_primes(bits, n, count)``: descending from 2^bits in steps of 2n,
  the primes q == 1 (mod 2n) below 2^bits (BASELINE.json configs; SURVEY.md
  Appendix A lists them).
- ``smallest_ntt_primes(bits, n, count)``: tests/test_util.hpp:16-26 (primes
  with exactly `bits` bits, smallest first).
- ``primes_with_bits(bits, count)``: tests/test_util.hpp:28-36.
"""
from __future__ import annotations

from functools import lru_cache


@lru_cache(maxsize=None)
def _is_prime(n):
    from oracle_lib import Oracle

    return Oracle().is_prime(n)


def largest_ntt_primes(bits, n, count):
    out = []
    c = ((1 << bits) - 1) // (2 * n) * (2 * n) + 1
    while len(out) < count and c > 2:
        if c < (1 << bits) and _is_prime(c):
            out.append(c)
        c -= 2 * n
    return out


def smallest_ntt_primes(bits, n, count):
    out = []
    two_n = 2 * n
    lo, hi = 1 << (bits - 1), 1 << bits
    c = ((lo - 1 + two_n - 1) // two_n) * two_n + 1
    while c < hi and len(out) < count:
        if c >= lo and _is_prime(c):
            out.append(c)
        c += two_n
    return out


def primes_with_bits(bits, count):
    out = []
    c = (1 << (bits - 1)) + 1
    while c < (1 << bits) and len(out) < count:
        if _is_prime(c):
            out.append(c)
        c += 2
    return out


SEED = 20260809  # bench.hpp:98 default seed


def config_seed(index):
    """Seed for BASELINE config `index` (1-based): index XOR the bench default seed."""
    return index ^ SEED


# BASELINE.json configs
def cfg1():
    return dict(n=4096, moduli=largest_ntt_primes(50, 4096, 1), npolys=1)


def cfg2_modulus():
    # largest prime < 2^60 (no NTT-friendliness needed): 2^60 - 93
    c = (1 << 60) - 1
    while not _is_prime(c):
        c -= 2
    return c


def cfg3():
    return dict(n=16384, moduli=largest_ntt_primes(50, 16384, 32), npolys=64)


def cfg4():
    return dict(n=65536, moduli=largest_ntt_primes(60, 65536, 24), npolys=16)


def cfg5():
    return dict(n=16384, moduli=largest_ntt_primes(50, 16384, 16), npolys=128)
