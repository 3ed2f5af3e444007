"""nttkit_b200 — B200 (sm_100a) negacyclic NTT and element-wise modular kernels.

A Python mirror of the reference's (nttkit, the portable restatement of Intel
HEXL, arXiv 2103.16400) operator interface for the hot path, over the C-ABI in
``include/nttkit_b200.h`` (``libnttkit_b200.so``, built in-tree by
``__graft_entry__.build()``). Names, argument meaning and error behaviour follow
the reference:

=============================  ===============================================
this module                    reference (/root/reference/proj/include/nttkit/)
=============================  ===============================================
``Modulus(q)``                 ``Modulus``            modarith.hpp:106-129
``NttTables(n, m, root, bs)``  ``NttTables``          ntt.hpp:206-247
``NttTables.forward``          ``NttTables::forward`` ntt.hpp:268-285
``NttTables.inverse``          ``NttTables::inverse`` ntt.hpp:289-306
``eltwise_mult_mod``           eltwise.hpp:180-188
``eltwise_mult_mod_int``       eltwise.hpp:137-154
``eltwise_mult_mod_float``     eltwise.hpp:158-175
``eltwise_fma_mod``            eltwise.hpp:263-271 (``z=None``: vector-scalar)
``eltwise_add_mod`` / ``_neg`` eltwise.hpp:47-70
``poly_mult_mod``              ring.hpp:28-43
``NTT``, ``EltwiseMultMod``,   HEXL names of the same calls
``EltwiseFMAMod``
``RnsNtt``                     one plan over many RNS limbs (batched, on device)
=============================  ===============================================

Buffers are numpy ``uint64`` arrays (host: copied to the GPU and back inside the
call, like the reference's blocking call) or ``torch.uint64`` CUDA tensors
(device: launched asynchronously on the current torch stream). Argument errors
raise ``ValueError`` carrying the reference's ``std::invalid_argument`` text.

There is no CPU fallback: if the library or a CUDA device is missing, calls
raise ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NK_LIB_PATH") or os.path.join(_HERE, "libnttkit_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "nttkit_b200.h")

u64 = C.c_uint64
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p

NK_ERR_CUDA = -100

_SIGS = {
    "nk_last_error": (C.c_char_p, []),
    "nk_version": (C.c_char_p, []),
    "nk_launch_count": (u64, []),
    "nk_debug_dump_to": (None, [vp]),
    "nk_debug_exact_only": (None, [C.c_int]),
    "nk_debug_block_kernel": (None, [C.c_int]),
    "nk_debug_butterflies": (C.c_int, [C.c_int, C.c_int, u64, u64, vp, vp, u64, vp, vp]),
    "nk_modulus": (C.c_int, [u64, C.POINTER(C.c_uint32), u64p]),
    "nk_minimal_primitive_root": (C.c_int, [u64, u64, u64p]),
    "nk_precompute_factor": (C.c_int, [u64, u64, C.c_int, u64p]),
    "nk_harvey_butterflies": (C.c_int, [C.c_int, u64, C.c_int, u64, u64, vp, vp, u64, vp, vp, C.c_int]),
    "nk_tables_host": (C.c_int, [u64, u64, u64p, C.c_int, u64p, u64p, u64p, u64p, u64p, u64p,
                                 u64p, C.POINTER(C.c_int)]),
    "nk_plan_create": (C.c_int, [C.POINTER(vp), C.c_int, u64, u64p, u64p, C.c_uint32, C.c_int]),
    "nk_plan_destroy": (None, [vp]),
    "nk_plan_info": (C.c_int, [vp, C.c_uint32, u64p, u64p, u64p, C.POINTER(C.c_int),
                               C.POINTER(C.c_uint32)]),
    "nk_ntt_forward": (C.c_int, [vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, u64, u64, vp]),
    "nk_ntt_inverse": (C.c_int, [vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, u64, u64, vp]),
    "nk_plan_eltwise_mult_mod": (C.c_int, [vp, vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32,
                                           u64, vp]),
    "nk_poly_mult_mod": (C.c_int, [vp, vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, vp]),
    "nk_eltwise_mult_mod": (C.c_int, [vp, vp, vp, u64, u64, u64, vp]),
    "nk_eltwise_mult_mod_int": (C.c_int, [vp, vp, vp, u64, u64, u64, vp]),
    "nk_eltwise_mult_mod_float": (C.c_int, [vp, vp, vp, u64, u64, u64, vp]),
    "nk_eltwise_fma_mod": (C.c_int, [vp, vp, u64, vp, u64, u64, u64, C.c_int, vp]),
    "nk_eltwise_add_mod": (C.c_int, [vp, vp, vp, u64, u64, vp]),
    "nk_eltwise_neg_mod": (C.c_int, [vp, vp, u64, u64, vp]),
    "nk_ntt_forward_host": (C.c_int, [vp, vp, vp, u64, C.c_uint32, C.c_uint32, C.c_uint32, u64,
                                      u64, vp]),
    "nk_ntt_inverse_host": (C.c_int, [vp, vp, vp, u64, C.c_uint32, C.c_uint32, C.c_uint32, u64,
                                      u64, vp]),
    "nk_poly_mult_mod_host": (C.c_int, [vp, vp, vp, vp, u64, C.c_uint32, C.c_uint32, C.c_uint32,
                                        vp]),
    "nk_eltwise_add_mod_host": (C.c_int, [vp, vp, vp, u64, u64, C.c_int, vp]),
    "nk_eltwise_neg_mod_host": (C.c_int, [vp, vp, u64, u64, C.c_int, vp]),
    "nk_eltwise_mult_mod_host": (C.c_int, [vp, vp, vp, u64, u64, u64, C.c_int, vp]),
    "nk_eltwise_mult_mod_int_host": (C.c_int, [vp, vp, vp, u64, u64, u64, C.c_int, vp]),
    "nk_eltwise_mult_mod_float_host": (C.c_int, [vp, vp, vp, u64, u64, u64, C.c_int, vp]),
    "nk_eltwise_fma_mod_host": (C.c_int, [vp, vp, u64, vp, u64, u64, u64, C.c_int, C.c_int, vp]),
}

_lib_handle = None


def lib():
    """Load libnttkit_b200.so (raises if it has not been built)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib_handle = h
    return _lib_handle


class CudaError(RuntimeError):
    pass


def _check(rc):
    if rc == 0:
        return
    msg = lib().nk_last_error().decode()
    if rc == NK_ERR_CUDA:
        raise CudaError(msg)
    raise ValueError(msg)


# ---------------------------------------------------------------------------
# buffer helpers
# ---------------------------------------------------------------------------
def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _dev_ptr(x):
    if x is None:
        return None
    import torch

    if not x.is_cuda:
        raise ValueError("device entry points need CUDA tensors")
    if x.dtype not in (torch.uint64, torch.int64):
        raise ValueError("tensors must be uint64 (or int64 bit patterns)")
    if not x.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return C.c_void_p(x.data_ptr())


def _stream_of(x):
    import torch

    return C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)


def _host_arr(x, name):
    a = np.asarray(x)
    if a.dtype != np.uint64:
        a = a.astype(np.uint64)
    return np.ascontiguousarray(a)


def _hp(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _host_out(result, like, what):
    """The result buffer of a host-buffer call: a fresh array like `like`, or
    the caller's array, which must be a C-contiguous numpy uint64 array of the
    same size (the library writes size * 8 bytes through its pointer)."""
    if result is None:
        return np.empty_like(like)
    if (not isinstance(result, np.ndarray) or result.dtype != np.uint64
            or not result.flags["C_CONTIGUOUS"] or not result.flags["WRITEABLE"]):
        raise ValueError("result must be a writeable C-contiguous numpy uint64 array")
    if result.size != like.size:
        raise ValueError(what)
    return result


def _same_numel(what, *xs):
    """Device calls: every tensor (None skipped) holds the same number of words."""
    ns = {x.numel() for x in xs if x is not None}
    if len(ns) > 1:
        raise ValueError(what)


def _np_u64_list(v):
    return np.ascontiguousarray(np.asarray(v, dtype=np.uint64).reshape(-1))


# ---------------------------------------------------------------------------
# host-only helpers
# ---------------------------------------------------------------------------
class Modulus:
    """Modulus(q) — modarith.hpp:106-129."""

    def __init__(self, q):
        bits = C.c_uint32()
        k = u64()
        _check(lib().nk_modulus(int(q), C.byref(bits), C.byref(k)))
        self._q, self._bits, self._k = int(q), bits.value, k.value

    def value(self):
        return self._q

    def bits(self):
        return self._bits

    def barrett_shift(self):
        return 63 + self._bits

    def barrett_factor(self):
        return self._k

    def __eq__(self, other):
        return isinstance(other, Modulus) and other._q == self._q

    def __repr__(self):
        return f"Modulus({self._q})"


def bit_reverse(i, log2n):
    """Reverse the low log2n bits of i (ntt.hpp:37-46)."""
    i, log2n = int(i), int(log2n)
    if not (0 <= log2n < 64 and (i == 0 if log2n == 0 else i >> log2n == 0)):
        raise ValueError("bit_reverse: index must have log2n bits")
    return int(format(i, f"0{log2n}b")[::-1], 2) if log2n else 0


def bit_reverse_permute(v):
    """In-place bit-reversal permutation of a power-of-two-length array (ntt.hpp:49-58)."""
    n = len(v)
    if n == 0 or n & (n - 1):
        raise ValueError("bit_reverse_permute: length must be a power of two")
    log2n = n.bit_length() - 1
    for i in range(n):
        j = bit_reverse(i, log2n)
        if i < j:
            v[i], v[j] = v[j], v[i]
    return v


def minimal_primitive_root(order, m):
    q = m.value() if isinstance(m, Modulus) else int(m)
    r = u64()
    _check(lib().nk_minimal_primitive_root(int(order), q, C.byref(r)))
    return r.value


class MultiplyFactor:
    """precompute_factor<bit_shift>(w, m) (modarith.hpp:168-183)."""

    def __init__(self, operand, m, bit_shift=64):
        q = m.value() if isinstance(m, Modulus) else int(m)
        p = u64()
        _check(lib().nk_precompute_factor(int(operand), q, int(bit_shift), C.byref(p)))
        self.operand, self.precon, self.bit_shift = int(operand), p.value, int(bit_shift)


def precompute_factor(w, m, bit_shift=64):
    return MultiplyFactor(w, m, bit_shift)


def _harvey(fwd, x0, x1, w, m):
    q = m.value() if isinstance(m, Modulus) else int(m)
    scalar = np.isscalar(x0)
    a = np.ascontiguousarray(np.atleast_1d(np.asarray(x0, dtype=np.uint64)))
    b = np.ascontiguousarray(np.atleast_1d(np.asarray(x1, dtype=np.uint64)))
    if a.size != b.size:
        raise ValueError("eltwise: operand lengths must match")
    y0, y1 = np.empty_like(a), np.empty_like(b)
    _check(lib().nk_harvey_butterflies(int(fwd), q, w.bit_shift, w.operand, w.precon, _hp(a), _hp(b),
                                       a.size, _hp(y0), _hp(y1), _device_of_default()))
    return (int(y0[0]), int(y1[0])) if scalar else (y0, y1)


def harvey_forward_butterfly(x0, x1, w, m):
    """harvey_forward_butterfly<B> (ntt.hpp:137-149), computed on the GPU;
    scalars or equal-length uint64 arrays; w a MultiplyFactor of width B."""
    return _harvey(True, x0, x1, w, m)


def harvey_inverse_butterfly(x0, x1, w, m):
    """harvey_inverse_butterfly<B> (ntt.hpp:154-166), computed on the GPU."""
    return _harvey(False, x0, x1, w, m)


def tables_host(n, q, root=None, bit_shift=0):
    """The NttTables precompute (host side of nk_plan_create), for parity checks."""
    arrs = [np.zeros(n, np.uint64) for _ in range(4)]
    psi, ninv, ninvp = u64(), u64(), u64()
    bs = C.c_int()
    rp = None if root is None else C.byref(u64(int(root)))
    _check(lib().nk_tables_host(int(n), int(q), rp, int(bit_shift), C.byref(psi),
                                *[a.ctypes.data_as(u64p) for a in arrs], C.byref(ninv),
                                C.byref(ninvp), C.byref(bs)))
    return dict(psi=psi.value, w=arrs[0], wp=arrs[1], wi=arrs[2], wip=arrs[3], ninv=ninv.value,
                ninvp=ninvp.value, bit_shift=bs.value)


def launch_count():
    return lib().nk_launch_count()


def set_exact_only(on):
    """Testing aid (nk_debug_exact_only): force the exact lazy arithmetic on
    every beta = 2^52 transform, including canonical-output ones."""
    lib().nk_debug_exact_only(1 if on else 0)


def debug_butterflies(policy, fwd, q, w, x0, x1):
    """Testing aid (nk_debug_butterflies): one butterfly per element pair of the
    int64 CUDA tensors x0, x1 in a kernel arithmetic policy; returns (y0, y1)."""
    import torch
    y0, y1 = torch.empty_like(x0), torch.empty_like(x1)
    _check(lib().nk_debug_butterflies(int(policy), int(bool(fwd)), int(q), int(w), _dev_ptr(x0),
                                      _dev_ptr(x1), x0.numel(), _dev_ptr(y0), _dev_ptr(y1)))
    return y0, y1


def set_block_kernel(which):
    """Testing aid (nk_debug_block_kernel): -1 = default (2), 0 = CTA-pair
    kernel, 1 = group-exchange kernel, 2 = two streams per thread, for
    16384-word blocks; 3 = defaults, but poly_mult_mod by the group-exchange
    single kernel;
    6 = defaults, but small batches of 2^11..2^13-word rows take the plain
    block kernel instead of the latency kernel."""
    lib().nk_debug_block_kernel(int(which))


# ---------------------------------------------------------------------------
# RNS plan: tables of many limbs resident on one device
# ---------------------------------------------------------------------------
class RnsNtt:
    """Negacyclic NTT tables for ``len(moduli)`` RNS limbs of length-n rows.

    Batched data is ``[npolys][nlimbs][n]`` uint64 (row = poly * nlimbs + limb).
    """

    def __init__(self, n, moduli, roots=None, bit_shift=0, device=None):
        mods = _np_u64_list(moduli)
        rts = None if roots is None else _np_u64_list(roots)
        if device is None:
            device = 0
            try:
                import torch

                if torch.cuda.is_available():
                    device = torch.cuda.current_device()
            except ImportError:
                pass
        h = vp()
        _check(lib().nk_plan_create(C.byref(h), int(device), int(n), mods.ctypes.data_as(u64p),
                                    None if rts is None else rts.ctypes.data_as(u64p),
                                    int(mods.size), int(bit_shift)))
        self._h = h
        self.n = int(n)
        self.nlimbs = int(mods.size)
        self.device = int(device)
        self.moduli = [int(x) for x in mods]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            try:
                lib().nk_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def info(self, limb=0):
        n, q, psi, nl = u64(), u64(), u64(), C.c_uint32()
        bs = C.c_int()
        _check(lib().nk_plan_info(self._h, limb, C.byref(n), C.byref(q), C.byref(psi),
                                  C.byref(bs), C.byref(nl)))
        return dict(n=n.value, q=q.value, psi=psi.value, bit_shift=bs.value, nlimbs=nl.value)

    def _rows(self, x, limb0, nlimbs):
        nl = self.nlimbs - limb0 if nlimbs is None else nlimbs
        total = x.numel() if _is_torch(x) else np.asarray(x).size
        if total % (self.n * nl):
            raise ValueError("transform: buffer length must equal n")
        return nl, total // (self.n * nl)

    def _transform(self, fwd, result, operand, fin, fout, limb0, nlimbs, stream):
        nl, npolys = self._rows(operand, limb0, nlimbs)
        if _is_torch(operand):
            if result.numel() != operand.numel():
                raise ValueError("transform: buffer length must equal n")
            st = _stream_of(operand) if stream is None else C.c_void_p(stream)
            fn = lib().nk_ntt_forward if fwd else lib().nk_ntt_inverse
            _check(fn(self._h, _dev_ptr(result), _dev_ptr(operand), limb0, nl, npolys, fin, fout, st))
            return result
        op = _host_arr(operand, "operand")
        out = _host_out(result, op, "transform: buffer length must equal n")
        fn = lib().nk_ntt_forward_host if fwd else lib().nk_ntt_inverse_host
        _check(fn(self._h, _hp(out), _hp(op), op.size, limb0, nl, npolys, fin, fout,
                  None if stream is None else C.c_void_p(stream)))
        return out

    def forward(self, result, operand, input_mod_factor=1, output_mod_factor=1, limb0=0,
                nlimbs=None, stream=None):
        return self._transform(True, result, operand, int(input_mod_factor),
                               int(output_mod_factor), limb0, nlimbs, stream)

    def inverse(self, result, operand, input_mod_factor=1, output_mod_factor=1, limb0=0,
                nlimbs=None, stream=None):
        return self._transform(False, result, operand, int(input_mod_factor),
                               int(output_mod_factor), limb0, nlimbs, stream)

    def poly_mult_mod(self, result, f, g, limb0=0, nlimbs=None, stream=None):
        nl, npolys = self._rows(f, limb0, nlimbs)
        if _is_torch(f):
            _same_numel("poly_mult_mod: operand lengths must equal n", f, g, result)
            st = _stream_of(f) if stream is None else C.c_void_p(stream)
            _check(lib().nk_poly_mult_mod(self._h, _dev_ptr(result), _dev_ptr(f), _dev_ptr(g),
                                          limb0, nl, npolys, st))
            return result
        fa, ga = _host_arr(f, "f"), _host_arr(g, "g")
        if fa.size != ga.size:
            raise ValueError("poly_mult_mod: operand lengths must equal n")
        out = _host_out(result, fa, "poly_mult_mod: operand lengths must equal n")
        _check(lib().nk_poly_mult_mod_host(self._h, _hp(out), _hp(fa), _hp(ga), fa.size, limb0, nl,
                                           npolys, None if stream is None else C.c_void_p(stream)))
        return out

    def eltwise_mult_mod(self, result, a, b, input_mod_factor=1, limb0=0, nlimbs=None,
                         stream=None):
        nl, npolys = self._rows(a, limb0, nlimbs)
        _same_numel("eltwise: operand lengths must match", a, b, result)
        st = _stream_of(a) if stream is None else C.c_void_p(stream)
        _check(lib().nk_plan_eltwise_mult_mod(self._h, _dev_ptr(result), _dev_ptr(a), _dev_ptr(b),
                                              limb0, nl, npolys, int(input_mod_factor), st))
        return result


class NttTables(RnsNtt):
    """NttTables(n, Modulus[, root][, bit_shift]) — ntt.hpp:206-247, one limb."""

    def __init__(self, n, m, root=None, bit_shift=None, device=None):
        q = m.value() if isinstance(m, Modulus) else int(m)
        if not isinstance(m, Modulus):
            Modulus(q)  # same first error as the reference
        super().__init__(n, [q], None if root is None else [root],
                         0 if bit_shift is None else bit_shift, device)
        self._m = Modulus(q)

    def size(self):
        return self.n

    def modulus(self):
        return self._m

    def root(self):
        return self.info()["psi"]

    def bit_shift(self):
        return self.info()["bit_shift"]

    # ntt.hpp:249-261 accessors: host copies of the tables the plan was built
    # from (nk_tables_host, bit for bit the reference's build_tables)
    def _host_tables(self):
        if getattr(self, "_ht", None) is None:
            info = self.info()
            self._ht = tables_host(self.n, self._m.value(), info["psi"], info["bit_shift"])
        return self._ht

    def log2_size(self):
        return self.n.bit_length() - 1

    def inv_root(self):
        return int(self._host_tables()["wi"][self.n // 2])  # psi^-1 at bit_reverse(1)

    def inv_size(self):
        t = self._host_tables()
        f = MultiplyFactor.__new__(MultiplyFactor)
        f.operand, f.precon, f.bit_shift = t["ninv"], t["ninvp"], t["bit_shift"]
        return f

    def root_powers_rev(self):
        return self._host_tables()["w"]

    def root_precons_rev(self):
        return self._host_tables()["wp"]

    def inv_root_powers_rev(self):
        return self._host_tables()["wi"]

    def inv_root_precons_rev(self):
        return self._host_tables()["wip"]

    def forward(self, result, operand, input_mod_factor, output_mod_factor, stream=None):
        self._check_len(result, operand)
        return super().forward(result, operand, input_mod_factor, output_mod_factor, stream=stream)

    def inverse(self, result, operand, input_mod_factor, output_mod_factor, stream=None):
        self._check_len(result, operand)
        return super().inverse(result, operand, input_mod_factor, output_mod_factor, stream=stream)

    def _check_len(self, result, operand):
        ln = (lambda x: x.numel()) if _is_torch(operand) else (lambda x: np.asarray(x).size)
        if ln(operand) != self.n or (result is not None and ln(result) != self.n):
            raise ValueError("transform: buffer length must equal n")


# ---------------------------------------------------------------------------
# element-wise
# ---------------------------------------------------------------------------
def _q_of(m):
    return m.value() if isinstance(m, Modulus) else int(m)


def _device_of_default():
    try:
        import torch

        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    except ImportError:
        return 0


def _eltwise_mult(path, result, a, b, m, input_mod_factor, stream):
    q = _q_of(m)
    dev_fn, host_fn = {
        "auto": ("nk_eltwise_mult_mod", "nk_eltwise_mult_mod_host"),
        "int": ("nk_eltwise_mult_mod_int", "nk_eltwise_mult_mod_int_host"),
        "float": ("nk_eltwise_mult_mod_float", "nk_eltwise_mult_mod_float_host"),
    }[path]
    if _is_torch(a):
        if not (a.numel() == b.numel() == result.numel()):
            raise ValueError("eltwise: operand lengths must match")
        st = _stream_of(a) if stream is None else C.c_void_p(stream)
        _check(getattr(lib(), dev_fn)(_dev_ptr(result), _dev_ptr(a), _dev_ptr(b), a.numel(), q,
                                      int(input_mod_factor), st))
        return result
    aa, bb = _host_arr(a, "a"), _host_arr(b, "b")
    if aa.size != bb.size:
        raise ValueError("eltwise: operand lengths must match")
    out = _host_out(result, aa, "eltwise: operand lengths must match")
    _check(getattr(lib(), host_fn)(_hp(out), _hp(aa), _hp(bb), aa.size, q, int(input_mod_factor),
                                   _device_of_default(), None if stream is None else C.c_void_p(stream)))
    return out


def eltwise_mult_mod(result, a, b, m, input_mod_factor=1, stream=None):
    """result[i] = a[i]*b[i] mod q; inputs in [0, input_mod_factor*q) (eltwise.hpp:180-188:
    the FP64 path for q < 2^50, the integer path otherwise)."""
    return _eltwise_mult("auto", result, a, b, m, input_mod_factor, stream)


def eltwise_mult_mod_int(result, a, b, m, input_mod_factor=1, stream=None):
    """The integer-Barrett path (eltwise.hpp:137-154); requires input_mod_factor*q < 2^63."""
    return _eltwise_mult("int", result, a, b, m, input_mod_factor, stream)


def eltwise_mult_mod_float(result, a, b, m, input_mod_factor=1, stream=None):
    """The FP64 path (eltwise.hpp:158-175); requires q < 2^50."""
    return _eltwise_mult("float", result, a, b, m, input_mod_factor, stream)


def eltwise_fma_mod(result, a, y, z, m, input_mod_factor=1, bit_shift=0, stream=None):
    """result[i] = (a[i]*y + z[i]) mod q; z=None is the vector-scalar multiply
    (eltwise.hpp:231-271). bit_shift 0 picks the width as the reference does."""
    q = _q_of(m)
    if _is_torch(a):
        if result.numel() != a.numel() or (z is not None and z.numel() != a.numel()):
            raise ValueError("eltwise: operand lengths must match")
        st = _stream_of(a) if stream is None else C.c_void_p(stream)
        _check(lib().nk_eltwise_fma_mod(_dev_ptr(result), _dev_ptr(a), int(y), _dev_ptr(z),
                                        a.numel(), q, int(input_mod_factor), int(bit_shift), st))
        return result
    aa = _host_arr(a, "a")
    zz = None if z is None else _host_arr(z, "z")
    if zz is not None and zz.size != aa.size:
        raise ValueError("eltwise: operand lengths must match")
    out = _host_out(result, aa, "eltwise: operand lengths must match")
    _check(lib().nk_eltwise_fma_mod_host(_hp(out), _hp(aa), int(y), _hp(zz), aa.size, q,
                                         int(input_mod_factor), int(bit_shift),
                                         _device_of_default(),
                                         None if stream is None else C.c_void_p(stream)))
    return out


def eltwise_add_mod(result, a, b, m, stream=None):
    """result[i] = (a[i] + b[i]) mod q for canonical inputs (eltwise.hpp:47-57)."""
    q = _q_of(m)
    if _is_torch(a):
        if a.numel() != b.numel() or result.numel() != a.numel():
            raise ValueError("eltwise: operand lengths must match")
        st = _stream_of(a) if stream is None else C.c_void_p(stream)
        _check(lib().nk_eltwise_add_mod(_dev_ptr(result), _dev_ptr(a), _dev_ptr(b), a.numel(), q, st))
        return result
    aa, bb = _host_arr(a, "a"), _host_arr(b, "b")
    if aa.size != bb.size:
        raise ValueError("eltwise: operand lengths must match")
    out = _host_out(result, aa, "eltwise: operand lengths must match")
    _check(lib().nk_eltwise_add_mod_host(_hp(out), _hp(aa), _hp(bb), aa.size, q, _device_of_default(),
                                         None if stream is None else C.c_void_p(stream)))
    return out


def eltwise_neg_mod(result, a, m, stream=None):
    """result[i] = (q - a[i]) mod q for canonical inputs (eltwise.hpp:60-70)."""
    q = _q_of(m)
    if _is_torch(a):
        if result.numel() != a.numel():
            raise ValueError("eltwise: operand lengths must match")
        st = _stream_of(a) if stream is None else C.c_void_p(stream)
        _check(lib().nk_eltwise_neg_mod(_dev_ptr(result), _dev_ptr(a), a.numel(), q, st))
        return result
    aa = _host_arr(a, "a")
    out = _host_out(result, aa, "eltwise: operand lengths must match")
    _check(lib().nk_eltwise_neg_mod_host(_hp(out), _hp(aa), aa.size, q, _device_of_default(),
                                         None if stream is None else C.c_void_p(stream)))
    return out


def poly_mult_mod(result, f, g, tables):
    """Negacyclic product via fwd(1,4) x2, mult(4), inv(1,1) — ring.hpp:28-43."""
    return tables.poly_mult_mod(result, f, g)


# ---------------------------------------------------------------------------
# HEXL names
# ---------------------------------------------------------------------------
class NTT(NttTables):
    """intel::hexl::NTT(degree, q[, root]) with ComputeForward / ComputeInverse."""

    def __init__(self, degree, q, root=None, device=None):
        super().__init__(degree, Modulus(q), root, None, device)

    def ComputeForward(self, result, operand, input_mod_factor, output_mod_factor):
        return self.forward(result, operand, input_mod_factor, output_mod_factor)

    def ComputeInverse(self, result, operand, input_mod_factor, output_mod_factor):
        return self.inverse(result, operand, input_mod_factor, output_mod_factor)


def EltwiseMultMod(result, operand1, operand2, n, modulus, input_mod_factor):
    if (operand1.numel() if _is_torch(operand1) else np.asarray(operand1).size) != n:
        raise ValueError("eltwise: operand lengths must match")
    return eltwise_mult_mod(result, operand1, operand2, modulus, input_mod_factor)


def EltwiseFMAMod(result, arg1, arg2, arg3, n, modulus, input_mod_factor):
    if (arg1.numel() if _is_torch(arg1) else np.asarray(arg1).size) != n:
        raise ValueError("eltwise: operand lengths must match")
    return eltwise_fma_mod(result, arg1, arg2, arg3, modulus, input_mod_factor)


__all__ = [
    "Modulus", "NttTables", "RnsNtt", "NTT", "eltwise_mult_mod", "eltwise_fma_mod",
    "eltwise_add_mod", "eltwise_neg_mod", "poly_mult_mod", "EltwiseMultMod", "EltwiseFMAMod",
    "minimal_primitive_root", "tables_host", "launch_count", "lib", "CudaError", "bit_reverse",
    "bit_reverse_permute",
]
