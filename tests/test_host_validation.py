"""Host-buffer result validation of the Python mirror (CPU): the library
writes size * 8 bytes through a result's pointer, so every host-buffer entry
point must reject results that are not writeable C-contiguous uint64 arrays of
the operands' size before any call reaches the C-ABI (no GPU needed)."""
import numpy as np
import pytest

Q60 = 1152921504606846883


def bad_results(n):
    base = np.zeros(2 * n, np.uint64)
    ro = np.zeros(n, np.uint64)
    ro.flags.writeable = False
    return {
        "uint32": np.zeros(n, np.uint32),
        "int64": np.zeros(n, np.int64),
        "reversed": np.zeros(n, np.uint64)[::-1],
        "strided": base[::2],
        "short": np.zeros(n - 1, np.uint64),
        "long": np.zeros(n + 1, np.uint64),
        "readonly": ro,
        "list": [0] * n,
    }


@pytest.mark.parametrize("kind", list(bad_results(8)))
def test_host_results_rejected(nk, kind):
    n = 8
    a = np.arange(n, dtype=np.uint64)
    b = np.arange(n, dtype=np.uint64) + 1
    r = bad_results(n)[kind]
    calls = [
        lambda: nk.eltwise_mult_mod(r, a, b, Q60, 1),
        lambda: nk.eltwise_mult_mod_int(r, a, b, Q60, 1),
        lambda: nk.eltwise_fma_mod(r, a, 3, b, Q60, 1),
        lambda: nk.eltwise_fma_mod(r, a, 3, None, Q60, 1),
        lambda: nk.eltwise_add_mod(r, a, b, Q60),
        lambda: nk.eltwise_neg_mod(r, a, Q60),
    ]
    for call in calls:
        with pytest.raises(ValueError):
            call()


def test_host_operand_lengths_rejected(nk):
    a = np.arange(8, dtype=np.uint64)
    with pytest.raises(ValueError, match="operand lengths must match"):
        nk.eltwise_mult_mod(None, a, a[:7], Q60, 1)
    with pytest.raises(ValueError, match="operand lengths must match"):
        nk.eltwise_fma_mod(None, a, 3, a[:7], Q60, 1)
    with pytest.raises(ValueError, match="operand lengths must match"):
        nk.eltwise_add_mod(None, a, a[:7], Q60)


def test_host_out_accepts_valid(nk):
    from paper_2103_16400_b200 import _host_out

    like = np.zeros(5, np.uint64)
    assert _host_out(None, like, "x").shape == (5,)
    r = np.zeros(5, np.uint64)
    assert _host_out(r, like, "x") is r
