"""CPU-side checks of the drop-in boundary (no GPU needed):

- libnttkit_b200.so loads and exports every entry point include/nttkit_b200.h
  declares;
- host-only entry points (Modulus, minimal root, table precompute) agree with
  the oracle and hence with the reference;
- argument errors carry the reference's std::invalid_argument messages and
  are reported before any device work;
- without a device, compute calls fail loudly (no CPU fallback);
- the C++ facade's argument checks (tests/cpp/facade_test --cpu).
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from primes import largest_ntt_primes, smallest_ntt_primes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "nttkit_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nk_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(nk):
    lib = C.CDLL(nk.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header(nk):
    assert set(declared_symbols()) <= set(nk._SIGS), set(declared_symbols()) - set(nk._SIGS)


@pytest.mark.parametrize("n,bits", [(4, 5), (8, 7), (64, 30), (1024, 50), (4096, 50), (2048, 60),
                                    (16384, 50), (256, 61)])
def test_host_tables_match_oracle(nk, oracle, n, bits):
    q = 17 if bits == 5 else (97 if bits == 7 else largest_ntt_primes(bits, n, 1)[0])
    mine = nk.tables_host(n, q)
    ref = oracle.tables(n, q)
    assert mine["psi"] == ref["psi"] and mine["bit_shift"] == ref["bit_shift"]
    assert mine["ninv"] == ref["ninv"] and mine["ninvp"] == ref["ninvp"]
    for k in ("w", "wp", "wi", "wip"):
        assert np.array_equal(mine[k], ref[k]), k


def test_host_tables_forced_width_and_root(nk, oracle):
    q = smallest_ntt_primes(49, 64, 1)[0]
    for bs in (52, 64):
        a, b = nk.tables_host(64, q, bit_shift=bs), oracle.tables(64, q, 0, bs)
        assert all(np.array_equal(a[k], b[k]) for k in ("w", "wp", "wi", "wip"))
    psi = oracle.minimal_primitive_root(128, q)
    root = pow(psi, 5, q)
    a, b = nk.tables_host(64, q, root=root), oracle.tables(64, q, root)
    assert a["psi"] == root and np.array_equal(a["w"], b["w"])


def test_modulus_and_roots(nk):
    m = nk.Modulus(17)
    assert (m.value(), m.bits(), m.barrett_shift(), m.barrett_factor()) == (17, 5, 68, (1 << 68) // 17)
    for bad in (0, 1, 2, 15, 1 << 62):
        with pytest.raises(ValueError, match=re.escape("Modulus: value must be a prime in [3, 2^62)")):
            nk.Modulus(bad)
    assert nk.minimal_primitive_root(8, 17) == 2
    assert nk.minimal_primitive_root(4, nk.Modulus(5)) == 2


ERRORS = [
    # (n, q, root, bit_shift) -> message of ntt.hpp:219-236
    ((4, 13, None, 0), "NttTables: q must satisfy q == 1 (mod 2n)"),
    ((3, 17, None, 0), "NttTables: n must be a power of two in [2, 2^20]"),
    ((1, 17, None, 0), "NttTables: n must be a power of two in [2, 2^20]"),
    ((1 << 21, 17, None, 0), "NttTables: n must be a power of two in [2, 2^20]"),
    ((4, 17, None, 48), "NttTables: accumulator width must be 52 or 64"),
    ((4, 17, 3, 0), "NttTables: root is not a primitive 2n'th root of unity"),
    ((4, 17, 0, 0), "NttTables: root is not a primitive 2n'th root of unity"),
]


@pytest.mark.parametrize("args,msg", ERRORS)
def test_table_errors(nk, args, msg):
    n, q, root, bs = args
    with pytest.raises(ValueError, match=re.escape(msg)):
        nk.tables_host(n, q, root=root, bit_shift=bs)
    # plan creation reports the same error before touching a device
    with pytest.raises(ValueError, match=re.escape(msg)):
        nk.RnsNtt(n, [q], roots=None if root is None else [root], bit_shift=bs)


def test_52bit_width_needs_small_modulus(nk):
    big = smallest_ntt_primes(52, 4, 1)[0]
    with pytest.raises(ValueError, match=re.escape("NttTables: 52-bit accumulator requires 4q < 2^52")):
        nk.tables_host(4, big, bit_shift=52)
    assert nk.tables_host(4, big, bit_shift=64)["bit_shift"] == 64


def test_factor_errors_before_device(nk):
    lib = nk.lib()
    cases = [
        (lib.nk_ntt_forward, 3, 1, "forward: input_mod_factor must be 1, 2 or 4"),
        (lib.nk_ntt_forward, 1, 2, "forward: output_mod_factor must be 1 or 4"),
        (lib.nk_ntt_inverse, 4, 1, "inverse: input_mod_factor must be 1 or 2"),
        (lib.nk_ntt_inverse, 1, 4, "inverse: output_mod_factor must be 1 or 2"),
    ]
    for fn, fin, fout, msg in cases:
        rc = fn(None, None, None, 0, 1, 1, fin, fout, None)
        assert rc == -7 - cases.index((fn, fin, fout, msg))
        assert lib.nk_last_error().decode() == msg


def test_eltwise_errors_before_device(nk):
    q50 = smallest_ntt_primes(50, 1, 1)[0]
    q62 = smallest_ntt_primes(62, 1, 1)[0]
    with pytest.raises(ValueError, match="input_mod_factor must be 1, 2 or 4"):
        nk.eltwise_mult_mod(None, np.zeros(8, np.uint64), np.zeros(8, np.uint64), q50, 3)
    with pytest.raises(ValueError, match=re.escape("requires input_mod_factor*q < 2^63")):
        nk.eltwise_mult_mod(None, np.zeros(8, np.uint64), np.zeros(8, np.uint64), q62, 4)
    with pytest.raises(ValueError, match="scalar must be < q"):
        nk.eltwise_fma_mod(None, np.zeros(4, np.uint64), q50, None, q50, 1)
    with pytest.raises(ValueError, match="input_mod_factor must be 1, 2, 4 or 8"):
        nk.eltwise_fma_mod(None, np.zeros(4, np.uint64), 1, None, q50, 3)
    with pytest.raises(ValueError, match=re.escape("requires q < 2^61")):
        nk.eltwise_fma_mod(None, np.zeros(4, np.uint64), 1, None, q62, 1)
    with pytest.raises(ValueError, match=re.escape("requires input_mod_factor*q < 2^BitShift")):
        nk.eltwise_fma_mod(None, np.zeros(4, np.uint64), 1, None, q50, 8, bit_shift=52)
    with pytest.raises(ValueError, match="operand lengths must match"):
        nk.eltwise_mult_mod(None, np.zeros(8, np.uint64), np.zeros(7, np.uint64), q50, 1)
    # the explicit paths carry their own checks (eltwise.hpp:144-146, 165-167)
    q60 = smallest_ntt_primes(60, 1, 1)[0]
    with pytest.raises(ValueError, match=re.escape("eltwise_mult_mod_float: requires q < 2^50")):
        nk.eltwise_mult_mod_float(None, np.zeros(8, np.uint64), np.zeros(8, np.uint64), q60, 1)
    with pytest.raises(ValueError, match=re.escape("eltwise_mult_mod_int: requires input_mod_factor*q < 2^63")):
        nk.eltwise_mult_mod_int(None, np.zeros(8, np.uint64), np.zeros(8, np.uint64), q62, 4)
    with pytest.raises(ValueError, match="input_mod_factor must be 1, 2 or 4"):
        nk.eltwise_mult_mod_float(None, np.zeros(8, np.uint64), np.zeros(8, np.uint64), q50, 8)


def test_no_cpu_fallback_without_device(nk):
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a device is present")
    except ImportError:
        pass
    with pytest.raises(nk.CudaError):
        nk.RnsNtt(4096, [1125899906826241])
    with pytest.raises(nk.CudaError):
        nk.eltwise_mult_mod(None, np.ones(8, np.uint64), np.ones(8, np.uint64), 17, 1)


def test_cpp_facade_argument_checks():
    exe = os.path.join(ROOT, "tests", "cpp", "facade_test")
    if not os.path.exists(exe):
        import __graft_entry__

        __graft_entry__.build_facade_test()
    out = subprocess.run([exe, "--cpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade cpu checks ok" in out.stdout


def test_precompute_factor_and_butterfly_checks(nk):
    """precompute_factor (modarith.hpp:176-183, test_modarith.cpp:195) and the
    public butterflies' argument checks (ntt.hpp:142-144,159-161), before any
    device work."""
    assert nk.precompute_factor(1, 17, 64).precon == 1085102592571150095
    assert nk.precompute_factor(3, 17, 52).precon == (3 << 52) // 17
    with pytest.raises(ValueError, match="operand must be < q"):
        nk.precompute_factor(17, 17, 64)
    q52 = smallest_ntt_primes(52, 1, 1)[0]
    with pytest.raises(ValueError, match=re.escape("requires q < beta/4")):
        nk.precompute_factor(1, q52, 52)
    w = nk.precompute_factor(5, 17, 64)
    with pytest.raises(ValueError, match="inputs must be < 4q"):
        nk.harvey_forward_butterfly(68, 0, w, 17)
    with pytest.raises(ValueError, match="inputs must be < 2q"):
        nk.harvey_inverse_butterfly(0, 34, w, 17)


def test_bit_reverse_helpers(nk):
    """ntt.hpp:37-58 (test_ntt.cpp BitReverse): the mirror's host helpers."""
    assert nk.bit_reverse(1, 3) == 4 and nk.bit_reverse(6, 3) == 3 and nk.bit_reverse(0, 0) == 0
    with pytest.raises(ValueError):
        nk.bit_reverse(8, 3)
    v = list(range(8))
    assert nk.bit_reverse_permute(v) == [0, 4, 2, 6, 1, 5, 3, 7]
    assert nk.bit_reverse_permute(v) == list(range(8))
    with pytest.raises(ValueError):
        nk.bit_reverse_permute([0] * 6)
    assert nk.minimal_primitive_root(8, 17) == 2 and nk.minimal_primitive_root(4, 5) == 2
