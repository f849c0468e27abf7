"""oracle -- TEST INFRASTRUCTURE ONLY.

Python (ctypes) access to the two CPU checkers of the B200 `lance_gemm` path:

* ``Oracle``: the plain-C restatement (``oracle/lance_oracle.c``), every
  function citing the reference file:line it restates.
* ``Reference``: the UNMODIFIED reference headers compiled in place
  (``oracle/_ref/libref_lance.so``, built by ``oracle/Makefile`` from
  ``/root/reference/proj/include``), exposing ``lance::lance_gemm``
  (engines.hpp:492-536), its stage functions and ``run_verify``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the timed CPU
baseline -- never as the thing measured for the GPU or shipped.  Parity of the
restatement is pinned against ``Reference`` and the golden vectors in
``tests/golden`` (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "liblance_oracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libref_lance.so")

PER_TILE, PER_POSITION, PER_TENSOR = 0, 1, 2


class OracleError(ValueError):
    """Mirrors std::invalid_argument thrown by the reference."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build() -> None:
    """Compile the oracle (and the reference shim when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


class _QP(ct.Structure):
    _fields_ = [("bits", ct.c_int), ("t_min", ct.c_float), ("t_max", ct.c_float),
                ("scale", ct.c_float)]


class _Spec(ct.Structure):
    _fields_ = [(n, ct.c_int) for n in ("n", "c", "h", "w", "k", "pad")]


class _Dump(ct.Structure):
    _fields_ = [("v", ct.c_void_p), ("u", ct.c_void_p), ("codes_a", ct.c_void_p),
                ("codes_w", ct.c_void_p), ("rowsum", ct.c_void_p), ("colsum", ct.c_void_p),
                ("acc", ct.c_void_p), ("params_a", ct.c_void_p), ("params_w", ct.c_void_p)]


@dataclass(frozen=True)
class Spec:
    n: int
    c: int
    h: int
    w: int
    k: int
    pad: int = 1

    @property
    def out_h(self):
        return self.h + 2 * self.pad - 2

    @property
    def out_w(self):
        return self.w + 2 * self.pad - 2

    @property
    def tiles(self):
        return ((self.out_h + 1) // 2) * ((self.out_w + 1) // 2)

    @property
    def rows(self):
        return self.n * self.tiles

    def tiles_m(self, m: int) -> int:
        """extract_tiles grid for tile side m (tensor.hpp:130-131)."""
        return ((self.out_h + m - 1) // m) * ((self.out_w + m - 1) // m)

    def rows_m(self, m: int) -> int:
        return self.n * self.tiles_m(m)


def _ptr(a):
    return a.ctypes.data_as(ct.c_void_p) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def params_to_array(qps) -> np.ndarray:
    """[16] x (bits, t_min, t_max, scale) as float32 [16, 4]."""
    return np.array([[q.bits, q.t_min, q.t_max, q.scale] for q in qps], dtype=np.float32)


class Oracle:
    """The C restatement (oracle/lance_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = ct.CDLL(path)
        lib.lo_last_error.restype = ct.c_char_p
        lib.lo_uniform_fill.argtypes = [ct.c_uint64, ct.c_void_p, ct.c_size_t]
        lib.lo_fit_params.argtypes = [ct.c_void_p, ct.c_size_t, ct.c_int, ct.POINTER(_QP)]
        lib.lo_quantize.argtypes = [ct.c_float, ct.POINTER(_QP)]
        lib.lo_quantize.restype = ct.c_uint8
        lib.lo_dequantize.argtypes = [ct.c_uint8, ct.POINTER(_QP)]
        lib.lo_dequantize.restype = ct.c_float
        lib.lo_affine_term.argtypes = [ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int,
                                       ct.POINTER(_QP), ct.POINTER(_QP)]
        lib.lo_affine_term.restype = ct.c_float
        for fn in ("lo_transform_input", "lo_transform_filter", "lo_transform_output",
                   "lo_transform_input4", "lo_transform_filter4", "lo_transform_output4"):
            getattr(lib, fn).argtypes = [ct.c_void_p, ct.c_void_p]
        lib.lo_lance_gemm_tiled.argtypes = [ct.POINTER(_Spec), ct.c_int, ct.c_int, ct.c_int,
                                            ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                            ct.POINTER(_QP), ct.POINTER(_Dump)]
        lib.lo_validate.argtypes = [ct.POINTER(_Spec), ct.c_int, ct.c_int, ct.c_int, ct.c_int]
        lib.lo_lance_gemm.argtypes = [ct.POINTER(_Spec), ct.c_int, ct.c_int, ct.c_int,
                                      ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                      ct.POINTER(_QP), ct.POINTER(_Dump)]
        lib.lo_direct_conv.argtypes = [ct.POINTER(_Spec), ct.c_void_p, ct.c_void_p, ct.c_void_p]
        self.lib = lib

    def _err(self, rc):
        if rc:
            raise OracleError(rc, self.lib.lo_last_error().decode())

    # -- fixtures ---------------------------------------------------------
    def uniform(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float32)
        self.lib.lo_uniform_fill(seed, _ptr(out), count)
        return out

    def layer(self, spec: Spec, seed: int):
        """x then w from one UniformSource stream (bench.hpp:129-133)."""
        nx = spec.n * spec.h * spec.w * spec.c
        nw = spec.k * 9 * spec.c
        s = self.uniform(seed, nx + nw)
        return (s[:nx].reshape(spec.n, spec.h, spec.w, spec.c),
                s[nx:].reshape(spec.k, 3, 3, spec.c))

    # -- primitives -------------------------------------------------------
    def transform_input(self, d):
        d = _f32(d).reshape(16)
        v = np.empty(16, np.float32)
        self.lib.lo_transform_input(_ptr(d), _ptr(v))
        return v.reshape(4, 4)

    def transform_filter(self, g):
        g = _f32(g).reshape(9)
        u = np.empty(16, np.float32)
        self.lib.lo_transform_filter(_ptr(g), _ptr(u))
        return u.reshape(4, 4)

    def transform_output(self, m):
        m = _f32(m).reshape(16)
        s = np.empty(4, np.float32)
        self.lib.lo_transform_output(_ptr(m), _ptr(s))
        return s.reshape(2, 2)

    # F(4x4,3x3) extension (Appendix D basis; not in the reference)
    def transform_input4(self, d):
        d = _f32(d).reshape(36)
        v = np.empty(36, np.float32)
        self.lib.lo_transform_input4(_ptr(d), _ptr(v))
        return v.reshape(6, 6)

    def transform_filter4(self, g):
        g = _f32(g).reshape(9)
        u = np.empty(36, np.float32)
        self.lib.lo_transform_filter4(_ptr(g), _ptr(u))
        return u.reshape(6, 6)

    def transform_output4(self, m):
        m = _f32(m).reshape(36)
        s = np.empty(16, np.float32)
        self.lib.lo_transform_output4(_ptr(m), _ptr(s))
        return s.reshape(4, 4)

    def fit_params(self, values, bits):
        v = _f32(values).ravel()
        qp = _QP()
        self._err(self.lib.lo_fit_params(_ptr(v), v.size, bits, ct.byref(qp)))
        return qp

    @staticmethod
    def qparams(bits, t_min, t_max, scale):
        return _QP(bits, t_min, t_max, scale)

    def quantize(self, x, qp) -> int:
        return int(self.lib.lo_quantize(float(x), ct.byref(qp)))

    def dequantize(self, code, qp) -> float:
        return float(self.lib.lo_dequantize(int(code), ct.byref(qp)))

    def affine_term(self, dot, a_sum, b_sum, depth, pa, pb) -> float:
        return float(self.lib.lo_affine_term(dot, a_sum, b_sum, depth, ct.byref(pa), ct.byref(pb)))

    def validate(self, spec: Spec, bits_w=8, bits_i=8, gran=PER_POSITION, mode_gemm=True):
        s = _Spec(spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad)
        self._err(self.lib.lo_validate(ct.byref(s), bits_w, bits_i, gran, int(mode_gemm)))

    # -- the path ---------------------------------------------------------
    def lance_gemm(self, spec: Spec, x, w, bits_w=8, bits_i=8, gran=PER_POSITION,
                   in_params=None, dump=False, tile_m=2):
        """lance_gemm (engines.hpp:492-536); tile_m=4 is the F(4x4,3x3)
        extension (36 positions in every dump)."""
        x = _f32(x)
        w = _f32(w)
        s = _Spec(spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad)
        y = np.empty((spec.n, spec.out_h, spec.out_w, spec.k), np.float32)
        M, C, K = spec.rows_m(tile_m), spec.c, spec.k
        NP = (tile_m + 2) ** 2
        d = None
        bufs = {}
        if dump:
            bufs = dict(
                v=np.empty((NP, M, C), np.float32), u=np.empty((NP, C, K), np.float32),
                codes_a=np.empty((NP, M, C), np.uint8), codes_w=np.empty((NP, C, K), np.uint8),
                rowsum=np.empty((NP, M), np.int32), colsum=np.empty((NP, K), np.int32),
                acc=np.empty((NP, M, K), np.int32))
            pa = (_QP * NP)()
            pw = (_QP * NP)()
            d = _Dump(*(_ptr(bufs[k]) for k in ("v", "u", "codes_a", "codes_w", "rowsum",
                                                 "colsum", "acc")),
                      ct.cast(pa, ct.c_void_p), ct.cast(pw, ct.c_void_p))
        ip = None
        if in_params is not None:
            ip = (_QP * NP)(*[_QP(int(r[0]), r[1], r[2], r[3]) for r in np.asarray(in_params)])
        rc = self.lib.lo_lance_gemm_tiled(ct.byref(s), tile_m, bits_w, bits_i, gran, _ptr(x),
                                          _ptr(w), _ptr(y), ip,
                                          ct.byref(d) if d is not None else None)
        self._err(rc)
        if not dump:
            return y
        bufs["params_a"] = params_to_array(pa)
        bufs["params_w"] = params_to_array(pw)
        return y, bufs

    def direct_conv(self, spec: Spec, x, w):
        x = _f32(x)
        w = _f32(w)
        s = _Spec(spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad)
        y = np.empty((spec.n, spec.out_h, spec.out_w, spec.k), np.float32)
        self.lib.lo_direct_conv(ct.byref(s), _ptr(x), _ptr(w), _ptr(y))
        return y


class Reference:
    """The reference headers compiled in place (oracle/_ref/libref_lance.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (reference tree absent?)")
        lib = ct.CDLL(path)
        lib.ref_last_error.restype = ct.c_char_p
        lib.ref_uniform_fill.argtypes = [ct.c_uint64, ct.c_void_p, ct.c_size_t]
        ints = [ct.c_int] * 6
        lib.ref_lance_gemm.argtypes = ints + [ct.c_int] * 4 + [ct.c_void_p] * 3
        lib.ref_lance_faithful.argtypes = ints + [ct.c_int] * 3 + [ct.c_void_p] * 3
        lib.ref_stage_dump.argtypes = ints + [ct.c_int] * 3 + [ct.c_void_p] * 11
        lib.ref_time_lance_gemm.argtypes = ints + [ct.c_int, ct.c_uint64, ct.c_int,
                                                   ct.POINTER(ct.c_double),
                                                   ct.POINTER(ct.c_double)]
        lib.ref_run_verify.argtypes = [ct.c_char_p, ct.c_size_t]
        lib.ref_set_threads.argtypes = [ct.c_int]
        lib.ref_write_lten.argtypes = [ct.c_char_p] + [ct.c_int] * 4 + [ct.c_void_p]
        lib.ref_read_lten.argtypes = [ct.c_char_p, ct.c_void_p, ct.c_void_p, ct.c_size_t]
        self.lib = lib

    def _err(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())

    def set_threads(self, n: int):
        self.lib.ref_set_threads(n)

    def uniform(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float32)
        self.lib.ref_uniform_fill(seed, _ptr(out), count)
        return out

    def lance_gemm(self, spec: Spec, x, w, bits_w=8, bits_i=8, gran=PER_POSITION, mode_gemm=True):
        x = _f32(x)
        w = _f32(w)
        y = np.empty((spec.n, spec.out_h, spec.out_w, spec.k), np.float32)
        rc = self.lib.ref_lance_gemm(spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad, bits_w,
                                     bits_i, gran, int(mode_gemm), _ptr(x), _ptr(w), _ptr(y))
        self._err(rc)
        return y

    def lance_faithful(self, spec: Spec, x, w, bits_w=8, bits_i=8, gran=PER_POSITION):
        x = _f32(x)
        w = _f32(w)
        y = np.empty((spec.n, spec.out_h, spec.out_w, spec.k), np.float32)
        rc = self.lib.ref_lance_faithful(spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad,
                                         bits_w, bits_i, gran, _ptr(x), _ptr(w), _ptr(y))
        self._err(rc)
        return y

    def stage_dump(self, spec: Spec, x, w, bits_w=8, bits_i=8, gran=PER_POSITION):
        x = _f32(x)
        w = _f32(w)
        M, C, K = spec.rows, spec.c, spec.k
        b = dict(v=np.empty((16, M, C), np.float32), u=np.empty((16, C, K), np.float32),
                 codes_a=np.empty((16, M, C), np.uint8), codes_w=np.empty((16, C, K), np.uint8),
                 params_a=np.empty((16, 4), np.float32), params_w=np.empty((16, 4), np.float32),
                 acc=np.empty((16, M, K), np.int32), rowsum=np.empty((16, M), np.int32),
                 colsum=np.empty((16, K), np.int32))
        rc = self.lib.ref_stage_dump(spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad, bits_w,
                                     bits_i, gran, _ptr(x), _ptr(w),
                                     *(_ptr(b[k]) for k in ("v", "u", "codes_a", "codes_w",
                                                             "params_a", "params_w", "acc",
                                                             "rowsum", "colsum")))
        self._err(rc)
        return b

    def time_lance_gemm(self, spec: Spec, threads: int, seed: int = 42, reps: int = 3):
        med = ct.c_double()
        mn = ct.c_double()
        rc = self.lib.ref_time_lance_gemm(spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad,
                                          threads, seed, reps, ct.byref(med), ct.byref(mn))
        self._err(rc)
        return med.value, mn.value

    def write_lten(self, path: str, t):
        t = _f32(t)
        n, h, w, c = t.shape
        self._err(self.lib.ref_write_lten(path.encode(), n, h, w, c, _ptr(t)))

    def read_lten(self, path: str):
        dims = np.zeros(4, np.int32)
        self._err(self.lib.ref_read_lten(path.encode(), _ptr(dims), None, 0))
        out = np.empty(tuple(int(d) for d in dims), np.float32)
        self._err(self.lib.ref_read_lten(path.encode(), _ptr(dims), _ptr(out), out.size))
        return out

    def run_verify(self):
        buf = ct.create_string_buffer(1 << 16)
        rc = self.lib.ref_run_verify(buf, len(buf))
        return rc == 0, buf.value.decode()


def reference_available() -> bool:
    return os.path.exists(REF_SO)
