"""Python mirror of the reference operator API for the lance_gemm path.

Names, fields, defaults and error behaviour follow
/root/reference/proj/include/lance/:

* ``ConvSpec``     engines.hpp:33-54   (r = s = 3, stride = 1 fixed)
* ``LanceConfig``  engines.hpp:60-80   (defaults bits 8/8, PerTile, Faithful)
* ``QuantParams``  quant.hpp:27-37
* ``Granularity``  quant.hpp:44,  ``LanceMode`` engines.hpp:56
* ``lance_gemm(x, w, spec, cfg) -> y``  engines.hpp:492-536 (host arrays)
* ``LanceConv``    device-resident plan: filters prepared once per layer (K2),
  ``forward`` runs K0 -> K1 -> K3/K4 on CUDA tensors.

Errors: ``std::invalid_argument`` maps to ``ValueError`` (``LanceError``) with
the reference's message; CUDA failures raise ``RuntimeError``.  There is no
CPU fallback: without an sm_100 device every entry point raises.
"""
from __future__ import annotations

import ctypes as ct
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib


class LanceError(ValueError):
    """std::invalid_argument from the reference (spec/config/shape/NaN)."""


class LanceNaNError(LanceError):
    """fit_params: NaN in values (quant.hpp:62)."""


class LanceDeviceError(RuntimeError):
    """CUDA failure or no sm_100 device (the path has no CPU fallback)."""


class Granularity(enum.IntEnum):
    PerTile = 0
    PerPosition = 1
    PerTensor = 2


class LanceMode(enum.IntEnum):
    Faithful = 0
    Gemm = 1


@dataclass
class ConvSpec:
    n: int = 1
    c: int = 1
    h: int = 1
    w: int = 1
    k: int = 1
    pad: int = 0
    r = 3
    s = 3
    stride = 1

    def out_h(self) -> int:
        return self.h + 2 * self.pad - self.r + 1

    def out_w(self) -> int:
        return self.w + 2 * self.pad - self.s + 1

    def tiles_h(self) -> int:
        return (self.out_h() + 1) // 2

    def tiles_w(self) -> int:
        return (self.out_w() + 1) // 2

    def tiles_per_image(self) -> int:
        return self.tiles_h() * self.tiles_w()

    def validate(self) -> None:
        cfg = LanceConfig(granularity=Granularity.PerPosition, mode=LanceMode.Gemm)
        _check(_lib.lib().lance_validate(ct.byref(self._c()), ct.byref(cfg._c())))

    def _c(self) -> _lib.CSpec:
        return _lib.CSpec(self.n, self.c, self.h, self.w, self.k, self.pad)


@dataclass
class LanceConfig:
    bits_w: int = 8
    bits_i: int = 8
    granularity: Granularity = Granularity.PerTile
    mode: LanceMode = LanceMode.Faithful

    def _c(self) -> _lib.CConfig:
        return _lib.CConfig(self.bits_w, self.bits_i, int(self.granularity), int(self.mode))


@dataclass
class QuantParams:
    bits: int = 8
    t_min: float = 0.0
    t_max: float = 0.0
    scale: float = 0.0

    def max_code(self) -> int:
        return (1 << self.bits) - 1


def _check(rc: int) -> None:
    if rc == _lib.LANCE_OK:
        return
    msg = _lib.lib().lance_last_error().decode()
    if rc == _lib.LANCE_ERR_NAN:
        raise LanceNaNError(msg)
    if rc == _lib.LANCE_ERR_INVALID_ARGUMENT:
        raise LanceError(msg)
    raise LanceDeviceError(f"{_lib.lib().lance_status_string(rc).decode()}: {msg}")


def validate(spec: ConvSpec, cfg: LanceConfig) -> None:
    """The checks lance_gemm performs before any work (engines.hpp:493-499)."""
    _check(_lib.lib().lance_validate(ct.byref(spec._c()), ct.byref(cfg._c())))


def winograd_multiply_count(spec: ConvSpec) -> int:
    return int(_lib.lib().lance_winograd_multiply_count(ct.byref(spec._c())))


def winograd_multiply_count_tiled(spec: ConvSpec, tile_m: int) -> int:
    """(m+2)^2 * tiles * N * C * K for tile side m (2 or 4)."""
    return int(_lib.lib().lance_winograd_multiply_count_tiled(ct.byref(spec._c()), int(tile_m)))


def direct_multiply_count(spec: ConvSpec) -> int:
    return int(_lib.lib().lance_direct_multiply_count(ct.byref(spec._c())))


def uniform_floats(count: int, seed: int) -> np.ndarray:
    """lance::uniform_floats (rng.hpp:50-54): UniformSource(seed) stream."""
    out = np.empty(count, np.float32)
    _lib.lib().lance_uniform_fill(seed, out.ctypes.data, count)
    return out


def _host_f32(a, shape, name):
    """check_layer's dims check (engines.hpp:84-91): a 4-D array must have
    exactly the spec's shape (an NCHW array or a [K,C,3,3] filter bank with the
    right element count is rejected); a flat 1-D array of the right size is
    accepted as raw NHWC / KRSC storage."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim == 1 and a.size == int(np.prod(shape)):
        return a
    if tuple(a.shape) != tuple(shape):
        raise LanceError(f"{name} dims do not match spec")
    return a


def lance_gemm(x, w, spec: ConvSpec, cfg: LanceConfig, out: np.ndarray | None = None,
               tile_m: int = 2):
    """lance::lance_gemm (engines.hpp:492-536) on host arrays.

    x: [N][H][W][C] float32 (NHWC), w: [K][3][3][C] float32 (KRSC).
    Returns y: [N][OH][OW][K] float32.  Runs on the current CUDA device.
    tile_m=4 selects the F(4x4,3x3) extension (not in the reference).
    """
    L = _lib.lib()
    cs, cc = spec._c(), cfg._c()
    _check(L.lance_validate(ct.byref(cs), ct.byref(cc)))
    x = _host_f32(x, (spec.n, spec.h, spec.w, spec.c), "input tensor")
    w = _host_f32(w, (spec.k, 3, 3, spec.c), "filter")
    shape = (spec.n, spec.out_h(), spec.out_w(), spec.k)
    y = out if out is not None else np.empty(shape, np.float32)
    if y.dtype != np.float32 or not y.flags.c_contiguous or y.size != int(np.prod(shape)):
        raise LanceError("output buffer does not match spec")
    _check(L.lance_gemm_host_tiled(ct.byref(cs), ct.byref(cc), int(tile_m), x.ctypes.data,
                                   w.ctypes.data, y.ctypes.data))
    return y.reshape(shape)


def _stream_ptr(stream):
    if stream is None:
        import torch
        return ct.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ct.c_void_p(stream)
    return ct.c_void_p(stream.cuda_stream)


class LanceConv:
    """One layer on one device: the reference's lance_gemm split into a
    once-per-layer filter preparation and a per-batch forward.

    Tensors are torch CUDA tensors (torch is used only for device memory and
    streams); every kernel is the in-tree sm_100a library.
    """

    def __init__(self, spec: ConvSpec, cfg: LanceConfig, device: int = 0, tile_m: int = 2,
                 layout: str = "nhwc"):
        """tile_m=2: the reference F(2x2,3x3) path; tile_m=4: the F(4x4,3x3)
        extension (36 positions in params / dumps).  layout="nchw" reads x as
        [N, C, H, W] (north-star option: a staging transpose on the device,
        then the NHWC kernels; y stays NHWC, the reference layout)."""
        self.spec = spec
        self.cfg = cfg
        self.device = device
        self.tile_m = int(tile_m)
        if layout not in ("nhwc", "nchw"):
            raise LanceError("layout must be 'nhwc' or 'nchw'")
        self.layout = layout
        self._plan = ct.c_void_p()
        L = _lib.lib()
        _check(L.lance_plan_create_tiled(ct.byref(spec._c()), ct.byref(cfg._c()), self.tile_m,
                                         device, ct.byref(self._plan)))
        if layout == "nchw":
            rc = L.lance_plan_set_input_layout(self._plan, 1)
            if rc:
                self.close()
                _check(rc)
        self.positions = int(L.lance_plan_positions(self._plan))
        self._acc = None
        self._bias = None

    def close(self):
        if self._plan:
            _lib.lib().lance_plan_destroy(self._plan)
            self._plan = ct.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def rows(self) -> int:
        m = self.tile_m
        s = self.spec
        return s.n * ((s.out_h() + m - 1) // m) * ((s.out_w() + m - 1) // m)

    @property
    def device_bytes(self) -> int:
        return int(_lib.lib().lance_plan_device_bytes(self._plan))

    @property
    def input_shape(self):
        s = self.spec
        return (s.n, s.c, s.h, s.w) if self.layout == "nchw" else (s.n, s.h, s.w, s.c)

    def _check_tensor(self, t, shape, name):
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32
                and t.is_contiguous()):
            raise LanceError(f"{name} must be a contiguous float32 CUDA tensor of shape {shape}")
        # exact shape (engines.hpp:84-91); a flat 1-D tensor is raw NHWC / KRSC storage
        if not (tuple(t.shape) == tuple(shape) or (t.dim() == 1 and t.numel() == int(np.prod(shape)))):
            raise LanceError(f"{name} dims do not match spec: got {tuple(t.shape)}, expected {tuple(shape)}")

    def set_filters(self, w, stream=None):
        """K2: G g G^T + per-position quantisation (engines.hpp:215-233)."""
        s = self.spec
        self._check_tensor(w, (s.k, 3, 3, s.c), "filter")
        _check(_lib.lib().lance_plan_set_filters(self._plan, ct.c_void_p(w.data_ptr()),
                                                 _stream_ptr(stream)))

    def set_epilogue(self, bias=None, relu: bool = False, pool: bool = False):
        """Optional fused bias + ReLU (north-star extension) and fused 2x2 /
        stride-2 max-pool (layer-stack option, F(2x2) only): with pool=True
        the forward writes [N, OH/2, OW/2, K]."""
        if bias is not None:
            self._check_tensor(bias, (self.spec.k,), "bias")
        self._bias = bias
        L = _lib.lib()
        _check(L.lance_plan_set_epilogue(
            self._plan, ct.c_void_p(bias.data_ptr()) if bias is not None else None, int(relu)))
        _check(L.lance_plan_set_epilogue_pool(self._plan, int(bool(pool))))
        self.pool = bool(pool)

    @property
    def out_shape(self):
        s = self.spec
        if getattr(self, "pool", False):
            return (s.n, s.out_h() // 2, s.out_w() // 2, s.k)
        return (s.n, s.out_h(), s.out_w(), s.k)

    def set_acc_dump(self, acc):
        """Also write the raw int32 accumulators [positions][M][K] on later forwards."""
        import torch
        if acc is not None:
            if not (acc.is_cuda and acc.dtype == torch.int32 and acc.is_contiguous()
                    and acc.numel() == self.positions * self.rows * self.spec.k):
                raise LanceError("acc dump must be int32 CUDA [positions][M][K]")
        self._acc = acc
        _check(_lib.lib().lance_plan_set_acc_dump(
            self._plan, ct.c_void_p(acc.data_ptr()) if acc is not None else None))

    def ranges(self, x, out=None, stream=None):
        """K0 only: this batch's fitted per-position ranges as a float32 CUDA
        tensor [2P + 1] = [-t_min, t_max, nan] -- the layout one element-wise
        MAX all-reduce combines across batch shards (global-fit mode,
        engines.hpp:157-165)."""
        import torch
        s = self.spec
        self._check_tensor(x, self.input_shape, "input tensor")
        n = 2 * self.positions + 1
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=x.device)
        if not (out.is_cuda and out.dtype == torch.float32 and out.is_contiguous() and out.numel() == n):
            raise LanceError(f"ranges buffer must be a float32 CUDA tensor of {n} elements")
        _check(_lib.lib().lance_plan_ranges(self._plan, ct.c_void_p(x.data_ptr()),
                                            ct.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def forward(self, x, y=None, stream=None, params=None, ranges=None):
        """K0 -> K1 -> K3/K4.  Asynchronous on `stream`; call ``sync`` to
        surface a NaN error.  ``params`` (16 QuantParams) selects the
        static-params mode (no range pass); ``ranges`` (a reduced buffer from
        ``ranges()`` + a MAX all-reduce) fits the input params on the device
        from global ranges instead of this batch's (no host round trip)."""
        import torch
        s = self.spec
        self._check_tensor(x, self.input_shape, "input tensor")
        if y is None:
            y = torch.empty(self.out_shape, dtype=torch.float32, device=x.device)
        self._check_tensor(y, self.out_shape, "output")
        L = _lib.lib()
        if ranges is not None:
            if not (ranges.is_cuda and ranges.dtype == torch.float32 and ranges.is_contiguous()
                    and ranges.numel() == 2 * self.positions + 1):
                raise LanceError(f"ranges must be a float32 CUDA tensor of {2 * self.positions + 1} elements")
            _check(L.lance_plan_forward_ranges(self._plan, ct.c_void_p(ranges.data_ptr()),
                                               ct.c_void_p(x.data_ptr()), ct.c_void_p(y.data_ptr()),
                                               _stream_ptr(stream)))
        elif params is None:
            _check(L.lance_plan_forward(self._plan, ct.c_void_p(x.data_ptr()),
                                        ct.c_void_p(y.data_ptr()), _stream_ptr(stream)))
        else:
            if len(params) != self.positions:
                raise LanceError(f"static params: expected {self.positions} QuantParams")
            arr = (_lib.CQParams * self.positions)(
                *[_lib.CQParams(q.bits, q.t_min, q.t_max, q.scale) for q in params])
            _check(L.lance_plan_forward_static(self._plan, arr, ct.c_void_p(x.data_ptr()),
                                               ct.c_void_p(y.data_ptr()), _stream_ptr(stream)))
        return y

    def sync(self, stream=None):
        _check(_lib.lib().lance_plan_sync(self._plan, _stream_ptr(stream)))

    @property
    def last_launch_count(self) -> int:
        return int(_lib.lib().lance_plan_last_launch_count(self._plan))

    def stage_timing(self, enable: bool = True):
        """Record CUDA events between the K0 / K1 / K3-K4 launches of forwards."""
        _check(_lib.lib().lance_plan_stage_timing(self._plan, int(enable)))

    def read_stage_times(self):
        """(summed ms of [K0, K1, K3/K4], number of forwards) since enabling."""
        arr = (ct.c_double * 3)()
        n = ct.c_int()
        _check(_lib.lib().lance_plan_read_stage_times(self._plan, arr, ct.byref(n)))
        return [arr[0], arr[1], arr[2]], n.value

    def params(self):
        a = (_lib.CQParams * self.positions)()
        b = (_lib.CQParams * self.positions)()
        _check(_lib.lib().lance_plan_get_params(self._plan, a, b))
        conv = lambda arr: [QuantParams(q.bits, q.t_min, q.t_max, q.scale) for q in arr]
        return conv(a), conv(b)

    def debug_read(self, what: str) -> np.ndarray:
        s, M, P = self.spec, self.rows, self.positions
        table = {"codes_a": (_lib.DBG_CODES_A, (P, M, s.c), np.uint8),
                 "rowsum": (_lib.DBG_ROWSUM, (P, M), np.int32),
                 "codes_w": (_lib.DBG_CODES_W, (P, s.c, s.k), np.uint8),
                 "colsum": (_lib.DBG_COLSUM, (P, s.k), np.int32)}
        code, shape, dt = table[what]
        out = np.empty(shape, dt)
        _check(_lib.lib().lance_plan_debug_read(self._plan, code, out.ctypes.data, out.nbytes))
        return out


def params_array(qps) -> np.ndarray:
    """[P] QuantParams -> float32 [P, 4] (bits, t_min, t_max, scale)."""
    return np.array([[q.bits, q.t_min, q.t_max, q.scale] for q in qps], dtype=np.float32)
