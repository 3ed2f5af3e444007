"""ctypes loaders for the CPU checkers under oracle/ (TEST INFRASTRUCTURE ONLY).

- ``Oracle``: oracle/liboracle.so, the C restatement of the reference.
- ``Ref``:    oracle/_ref/libnttref.so, the unmodified reference headers behind
              a C shim (built here from /root/reference; the .so travels to the
              GPU box, the sources do not).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libnttref.so")

u64 = C.c_uint64
u64p = C.POINTER(C.c_uint64)


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(u64p)


def build_oracle():
    """Compile oracle/liboracle.so (and _ref when the reference is present)."""
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


class Oracle:
    _lib = None

    def __init__(self):
        if Oracle._lib is None:
            if not os.path.exists(ORACLE_SO):
                build_oracle()
            lib = C.CDLL(ORACLE_SO)
            sig = {
                "oc_is_prime": (C.c_int, [u64]),
                "oc_modulus": (C.c_int, [u64, C.POINTER(C.c_uint32), u64p]),
                "oc_barrett_reduce": (u64, [u64, u64, u64]),
                "oc_mul_mod": (u64, [u64, u64, u64]),
                "oc_pow_mod": (u64, [u64, u64, u64]),
                "oc_inv_mod": (u64, [u64, u64]),
                "oc_small_mod": (u64, [u64, u64, u64]),
                "oc_precompute_factor": (u64, [u64, u64, C.c_int]),
                "oc_bit_reverse": (u64, [u64, C.c_uint]),
                "oc_minimal_primitive_root": (u64, [u64, u64]),
                "oc_ntt_tables": (C.c_int, [u64, u64, u64, C.c_int, u64p, u64p, u64p, u64p,
                                            u64p, u64p, u64p, u64p]),
                "oc_ntt_forward": (C.c_int, [u64, u64p, C.c_uint32, C.c_int, u64p, u64p, u64,
                                             u64, u64, C.c_int]),
                "oc_ntt_inverse": (C.c_int, [u64, u64p, C.c_uint32, C.c_int, u64p, u64p, u64,
                                             u64, u64, C.c_int]),
                "oc_ntt_root": (C.c_int, [u64, u64, u64, C.c_int, C.c_int, u64p, u64p, u64, u64]),
                "oc_ntt_stages": (C.c_int, [u64, u64, C.c_int, u64p, u64, C.c_int]),
                "oc_reference_ntt": (C.c_int, [u64, u64, u64, C.c_int, u64p, u64p]),
                "oc_eltwise_add_mod": (C.c_int, [u64p, u64p, u64p, u64, u64]),
                "oc_eltwise_neg_mod": (C.c_int, [u64p, u64p, u64, u64]),
                "oc_eltwise_mult_mod": (C.c_int, [u64p, u64p, u64p, u64, u64, u64, C.c_int]),
                "oc_eltwise_fma_mod": (C.c_int, [u64p, u64p, u64, u64p, u64, u64, u64, C.c_int]),
                "oc_poly_mult_mod": (C.c_int, [u64, u64p, C.c_uint32, u64p, u64p, u64p, u64,
                                               C.c_int]),
                "oc_naive_negacyclic": (C.c_int, [u64, u64, u64p, u64p, u64p]),
                "oc_mt19937_64_fill": (None, [u64, u64p, u64, u64]),
                "oc_butterflies": (C.c_int, [C.c_int, u64, C.c_int, u64, u64p, u64p, u64, u64p, u64p]),
            }
            for name, (res, args) in sig.items():
                f = getattr(lib, name)
                f.restype = res
                f.argtypes = args
            Oracle._lib = lib
        self.lib = Oracle._lib

    # ---- scalar helpers ----
    def is_prime(self, n):
        return bool(self.lib.oc_is_prime(n))

    def modulus(self, q):
        bits = C.c_uint32()
        k = u64()
        rc = self.lib.oc_modulus(q, C.byref(bits), C.byref(k))
        if rc:
            raise ValueError("Modulus: value must be a prime in [3, 2^62)")
        return bits.value, k.value

    def butterflies(self, fwd, q, bs, w, x0, x1):
        """harvey_forward/inverse_butterfly (ntt.hpp:137-166) on element pairs."""
        x0 = np.ascontiguousarray(x0, np.uint64)
        x1 = np.ascontiguousarray(x1, np.uint64)
        y0, y1 = np.empty_like(x0), np.empty_like(x1)
        P = lambda a: a.ctypes.data_as(u64p)  # noqa: E731
        rc = self.lib.oc_butterflies(int(fwd), q, bs, w, P(x0), P(x1), x0.size, P(y0), P(y1))
        assert rc == 0
        return y0, y1

    def minimal_primitive_root(self, order, q):
        return self.lib.oc_minimal_primitive_root(order, q)

    def tables(self, n, q, root=0, bit_shift=0):
        arrs = [np.zeros(n, np.uint64) for _ in range(4)]
        psi, psii, ninv, ninvp = u64(), u64(), u64(), u64()
        bs = self.lib.oc_ntt_tables(n, q, root, bit_shift, C.byref(psi), C.byref(psii),
                                    *[_ptr(a) for a in arrs], C.byref(ninv), C.byref(ninvp))
        if bs < 0:
            raise ValueError(f"NttTables: invalid arguments ({bs})")
        return dict(psi=psi.value, psi_inv=psii.value, w=arrs[0], wp=arrs[1], wi=arrs[2],
                    wip=arrs[3], ninv=ninv.value, ninvp=ninvp.value, bit_shift=bs)

    # ---- transforms over [rows, n] with row r using moduli[r % len(moduli)] ----
    def _ntt(self, fn, n, moduli, x, fin, fout, bit_shift, threads):
        mod = np.ascontiguousarray(np.asarray(moduli, dtype=np.uint64).reshape(-1))
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.empty_like(x)
        rows = x.size // n
        rc = fn(n, _ptr(mod), mod.size, bit_shift, _ptr(out), _ptr(x), rows, fin, fout, threads)
        if rc:
            raise ValueError(f"transform: invalid arguments ({rc})")
        return out

    def _ntt_root(self, d, n, q, x, fin, fout, bit_shift, root):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.empty_like(x)
        rc = self.lib.oc_ntt_root(n, q, root, bit_shift, d, _ptr(out), _ptr(x), fin, fout)
        if rc:
            raise ValueError(f"transform: invalid arguments ({rc})")
        return out

    def forward(self, n, moduli, x, fin=1, fout=1, bit_shift=0, threads=1, root=0):
        if root:
            return self._ntt_root(0, n, int(moduli[0]), x, fin, fout, bit_shift, root)
        return self._ntt(self.lib.oc_ntt_forward, n, moduli, x, fin, fout, bit_shift, threads)

    def inverse(self, n, moduli, x, fin=1, fout=1, bit_shift=0, threads=1, root=0):
        if root:
            return self._ntt_root(1, n, int(moduli[0]), x, fin, fout, bit_shift, root)
        return self._ntt(self.lib.oc_ntt_inverse, n, moduli, x, fin, fout, bit_shift, threads)

    def reference_ntt(self, q, psi, a, direction):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        out = np.empty_like(a)
        self.lib.oc_reference_ntt(a.size, q, psi, 0 if direction == "forward" else 1,
                                  _ptr(a), _ptr(out))
        return out

    def eltwise_mult_mod(self, a, b, q, fin=1, path=0):
        a = np.ascontiguousarray(a, np.uint64)
        b = np.ascontiguousarray(b, np.uint64)
        r = np.empty_like(a)
        rc = self.lib.oc_eltwise_mult_mod(_ptr(r), _ptr(a), _ptr(b), a.size, q, fin, path)
        if rc:
            raise ValueError(f"eltwise_mult_mod: invalid arguments ({rc})")
        return r

    def eltwise_fma_mod(self, a, y, z, q, fin=1, bit_shift=0):
        a = np.ascontiguousarray(a, np.uint64)
        z = None if z is None else np.ascontiguousarray(z, np.uint64)
        r = np.empty_like(a)
        rc = self.lib.oc_eltwise_fma_mod(_ptr(r), _ptr(a), y, _ptr(z), a.size, q, fin, bit_shift)
        if rc:
            raise ValueError(f"eltwise_fma_mod: invalid arguments ({rc})")
        return r

    def eltwise_add_mod(self, a, b, q):
        a = np.ascontiguousarray(a, np.uint64)
        b = np.ascontiguousarray(b, np.uint64)
        r = np.empty_like(a)
        self.lib.oc_eltwise_add_mod(_ptr(r), _ptr(a), _ptr(b), a.size, q)
        return r

    def eltwise_neg_mod(self, a, q):
        a = np.ascontiguousarray(a, np.uint64)
        r = np.empty_like(a)
        self.lib.oc_eltwise_neg_mod(_ptr(r), _ptr(a), a.size, q)
        return r

    def poly_mult_mod(self, n, moduli, f, g, threads=1):
        mod = np.ascontiguousarray(np.asarray(moduli, dtype=np.uint64).reshape(-1))
        f = np.ascontiguousarray(f, np.uint64)
        g = np.ascontiguousarray(g, np.uint64)
        out = np.empty_like(f)
        rc = self.lib.oc_poly_mult_mod(n, _ptr(mod), mod.size, _ptr(out), _ptr(f), _ptr(g),
                                       f.size // n, threads)
        if rc:
            raise ValueError(f"poly_mult_mod: invalid arguments ({rc})")
        return out

    def naive_negacyclic(self, f, g, q):
        f = np.ascontiguousarray(f, np.uint64)
        g = np.ascontiguousarray(g, np.uint64)
        out = np.empty_like(f)
        self.lib.oc_naive_negacyclic(f.size, q, _ptr(f), _ptr(g), _ptr(out))
        return out

    def mt19937_64(self, seed, count, bound=0):
        out = np.empty(count, np.uint64)
        self.lib.oc_mt19937_64_fill(seed, _ptr(out), count, bound)
        return out


class Ref:
    """The reference's own code (oracle/_ref/libnttref.so)."""

    _lib = None

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        if Ref._lib is None:
            lib = C.CDLL(REF_SO)
            vp = C.c_void_p
            sig = {
                "ref_last_error": (C.c_char_p, []),
                "ref_hw_threads": (C.c_int, []),
                "ref_tables": (C.c_int, [u64, u64, u64, C.c_int, u64p, u64p, u64p, u64p, u64p,
                                         u64p, u64p, C.POINTER(C.c_int)]),
                "ref_ntt_forward": (C.c_int, [u64, u64p, C.c_uint32, C.c_int, u64p, u64p, u64,
                                              u64, u64, C.c_int]),
                "ref_ntt_inverse": (C.c_int, [u64, u64p, C.c_uint32, C.c_int, u64p, u64p, u64,
                                              u64, u64, C.c_int]),
                "ref_plan_create": (vp, [u64, u64p, C.c_uint32]),
                "ref_plan_destroy": (None, [vp]),
                "ref_plan_ntt": (C.c_int, [vp, C.c_int, u64p, u64p, u64, u64, u64, C.c_int]),
                "ref_plan_poly_mult": (C.c_int, [vp, u64p, u64p, u64p, u64, C.c_int]),
                "ref_eltwise_mult_mod": (C.c_int, [u64p, u64p, u64p, u64, u64, u64, C.c_int,
                                                   C.c_int]),
                "ref_eltwise_fma_mod": (C.c_int, [u64p, u64p, u64, u64p, u64, u64, u64, C.c_int,
                                                  C.c_int]),
                "ref_eltwise_add_mod": (C.c_int, [u64p, u64p, u64p, u64, u64]),
                "ref_eltwise_neg_mod": (C.c_int, [u64p, u64p, u64, u64]),
                "ref_reference_ntt": (C.c_int, [u64, u64, u64, C.c_int, u64p, u64p]),
                "ref_naive_negacyclic": (C.c_int, [u64, u64, u64p, u64p, u64p]),
                "ref_is_prime": (C.c_int, [u64]),
            }
            # added later in the round: bound only when the prebuilt library has it
            if hasattr(lib, "ref_butterflies"):
                sig["ref_butterflies"] = (C.c_int, [C.c_int, u64, C.c_int, u64, u64p, u64p, u64,
                                                    u64p, u64p])
            for name, (res, args) in sig.items():
                f = getattr(lib, name)
                f.restype = res
                f.argtypes = args
            Ref._lib = lib
        self.lib = Ref._lib

    def _check(self, rc):
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())

    def tables(self, n, q, root=0, bit_shift=0):
        arrs = [np.zeros(n, np.uint64) for _ in range(4)]
        psi, ninv, ninvp = u64(), u64(), u64()
        bs = C.c_int()
        self._check(self.lib.ref_tables(n, q, root, bit_shift, C.byref(psi),
                                        *[_ptr(a) for a in arrs], C.byref(ninv),
                                        C.byref(ninvp), C.byref(bs)))
        return dict(psi=psi.value, w=arrs[0], wp=arrs[1], wi=arrs[2], wip=arrs[3],
                    ninv=ninv.value, ninvp=ninvp.value, bit_shift=bs.value)

    def _ntt(self, fn, n, moduli, x, fin, fout, bit_shift, threads):
        mod = np.ascontiguousarray(np.asarray(moduli, dtype=np.uint64).reshape(-1))
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.empty_like(x)
        self._check(fn(n, _ptr(mod), mod.size, bit_shift, _ptr(out), _ptr(x), x.size // n, fin,
                       fout, threads))
        return out

    def forward(self, n, moduli, x, fin=1, fout=1, bit_shift=0, threads=1):
        return self._ntt(self.lib.ref_ntt_forward, n, moduli, x, fin, fout, bit_shift, threads)

    def inverse(self, n, moduli, x, fin=1, fout=1, bit_shift=0, threads=1):
        return self._ntt(self.lib.ref_ntt_inverse, n, moduli, x, fin, fout, bit_shift, threads)

    def butterflies(self, fwd, q, bs, w, x0, x1):
        x0 = np.ascontiguousarray(x0, np.uint64)
        x1 = np.ascontiguousarray(x1, np.uint64)
        y0, y1 = np.empty_like(x0), np.empty_like(x1)
        self._check(self.lib.ref_butterflies(int(fwd), q, bs, w, _ptr(x0), _ptr(x1), x0.size,
                                             _ptr(y0), _ptr(y1)))
        return y0, y1

    def eltwise_mult_mod(self, a, b, q, fin=1, path=0, threads=1):
        a = np.ascontiguousarray(a, np.uint64)
        b = np.ascontiguousarray(b, np.uint64)
        r = np.empty_like(a)
        self._check(self.lib.ref_eltwise_mult_mod(_ptr(r), _ptr(a), _ptr(b), a.size, q, fin,
                                                  path, threads))
        return r

    def eltwise_fma_mod(self, a, y, z, q, fin=1, bit_shift=0, threads=1):
        a = np.ascontiguousarray(a, np.uint64)
        z = None if z is None else np.ascontiguousarray(z, np.uint64)
        r = np.empty_like(a)
        self._check(self.lib.ref_eltwise_fma_mod(_ptr(r), _ptr(a), y, _ptr(z), a.size, q, fin,
                                                 bit_shift, threads))
        return r

    def eltwise_add_mod(self, a, b, q):
        a = np.ascontiguousarray(a, np.uint64)
        b = np.ascontiguousarray(b, np.uint64)
        r = np.empty_like(a)
        self._check(self.lib.ref_eltwise_add_mod(_ptr(r), _ptr(a), _ptr(b), a.size, q))
        return r

    def eltwise_neg_mod(self, a, q):
        a = np.ascontiguousarray(a, np.uint64)
        r = np.empty_like(a)
        self._check(self.lib.ref_eltwise_neg_mod(_ptr(r), _ptr(a), a.size, q))
        return r

    def poly_mult_mod(self, n, moduli, f, g, threads=1):
        mod = np.ascontiguousarray(np.asarray(moduli, dtype=np.uint64).reshape(-1))
        f = np.ascontiguousarray(f, np.uint64)
        g = np.ascontiguousarray(g, np.uint64)
        out = np.empty_like(f)
        p = self.lib.ref_plan_create(n, _ptr(mod), mod.size)
        if not p:
            raise ValueError(self.lib.ref_last_error().decode())
        try:
            self._check(self.lib.ref_plan_poly_mult(p, _ptr(out), _ptr(f), _ptr(g), f.size // n,
                                                    threads))
        finally:
            self.lib.ref_plan_destroy(p)
        return out

    def reference_ntt(self, q, psi, a, direction):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        out = np.empty_like(a)
        self._check(self.lib.ref_reference_ntt(a.size, q, psi,
                                               0 if direction == "forward" else 1,
                                               _ptr(a), _ptr(out)))
        return out

    def naive_negacyclic(self, f, g, q):
        f = np.ascontiguousarray(f, np.uint64)
        g = np.ascontiguousarray(g, np.uint64)
        out = np.empty_like(f)
        self._check(self.lib.ref_naive_negacyclic(f.size, q, _ptr(f), _ptr(g), _ptr(out)))
        return out
