"""Python host side of the MoBi linear layer over the C ABI.

Mirrors the reference's hot-path interface (router.hpp / bitplane.hpp / checkpoint.hpp):
the layer is built from the same objects the reference passes around -- a SliceStack
(codes, slice_bits, base QuantParams) plus a RouterState, or a checkpoint LayerRecord --
and exposes score / gate_hard / forward_elastic / permute_by_slice / calibrate_threshold
with the reference's argument meaning and error behaviour (ValueError for the reference's
std::invalid_argument).  torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import LayerDesc, OutDesc, check, lib

_i64, _i32, _f64 = C.c_int64, C.c_int32, C.c_double


def _stream_ptr(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def ratio_from_target_bits(target: float, slice_bits: Sequence[int]) -> float:
    """router.hpp:153-162."""
    if len(slice_bits) < 2:
        raise ValueError("ratio_from_target_bits: need at least one residual slice")
    b, r = float(slice_bits[0]), float(sum(slice_bits[1:]))
    if not (b <= target <= b + r):
        raise ValueError(f"ratio_from_target_bits: target {target:g} outside [{b:g},{b + r:g}]")
    return (target - b) / r


def avg_bits_from_masks(masks: torch.Tensor, slice_bits: Sequence[int], stream=None) -> float:
    """router.hpp:135-150 on device slice masks (bit e-1 <-> slice e): mobi_avg_bits."""
    m = masks.to(torch.uint8).contiguous()
    if not m.is_cuda:
        raise ValueError("avg_bits expects CUDA masks")
    sb = _arr(slice_bits, np.int32)
    out = _f64()
    check(lib().mobi_avg_bits(m.data_ptr() if m.numel() else None, m.numel(), sb.ctypes.data, sb.size, C.byref(out),
                              _stream_ptr(stream)))
    return out.value


class MobiLayer:
    """One MoBi linear layer resident on a B200."""

    def __init__(self, handle: int, slice_bits, out: int, inn: int, hidden: int, device: int):
        self._h = C.c_void_p(handle)
        self.slice_bits = list(slice_bits)
        self.out, self.inn, self.hidden, self.device = out, inn, hidden, device
        self.n_routed = len(self.slice_bits) - 1

    # ---------------- construction ----------------
    @classmethod
    def from_stack(cls, codes, slice_bits, scale, zero, group_size, w1, b1, w2, b2, device: int = 0):
        """From a SliceStack (codes [E,out,in] uint8, base scale/zero) + RouterState (w1 [in,h]...)."""
        codes = _arr(codes, np.uint8)
        E, out, inn = codes.shape
        return cls._create(out, inn, group_size, slice_bits, scale, zero, codes, None, 0, 0, w1, b1, w2, b2, device)

    @classmethod
    def from_device_stack(cls, codes: torch.Tensor, slice_bits, scale, zero, group_size, w1, b1, w2, b2):
        """From a SliceStack whose codes [E,out,in] uint8 already live on the GPU (e.g. decompose()'s
        output): validated and repacked on the device (mobi_layer_create_device)."""
        if not (codes.is_cuda and codes.dtype == torch.uint8 and codes.dim() == 3):
            raise ValueError("from_device_stack expects CUDA uint8 codes [E, out, in]")
        codes = codes.contiguous()
        E, out, inn = codes.shape
        return cls._create(out, inn, group_size, slice_bits, scale, zero, codes, None, 0, 0, w1, b1, w2, b2,
                           codes.device.index)

    @classmethod
    def from_record(cls, rec, device: int = 0):
        """From a checkpoint LayerRecord (merged-code bit-planes, checkpoint.hpp:30-74)."""
        planes = _arr(rec.planes, np.uint64)
        return cls._create(rec.rows, rec.cols, rec.group_size, rec.slice_bits, rec.base_scale, rec.base_zero,
                           None, planes, rec.plane_bits, planes.shape[2], rec.w1, rec.b1, rec.w2, rec.b2, device)

    @classmethod
    def from_stack_rows(cls, codes, slice_bits, scale, zero, group_size, w1, b1, w2, b2, row0: int, row1: int,
                        device: int = 0):
        """Column-parallel shard: weight rows [row0, row1) of the SliceStack + the full router
        (mobi_layer_create_rows)."""
        codes = _arr(codes, np.uint8)
        E, out, inn = codes.shape
        return cls._create(out, inn, group_size, slice_bits, scale, zero, codes, None, 0, 0, w1, b1, w2, b2, device,
                           rows=(row0, row1))

    @classmethod
    def _create(cls, out, inn, gs, slice_bits, scale, zero, codes, planes, plane_bits, wpr, w1, b1, w2, b2, device,
                rows=None):
        sb = _arr(slice_bits, np.int32)
        dev_codes = isinstance(codes, torch.Tensor)
        scale, zero = _arr(scale, np.float64), _arr(zero, np.float64)
        w1, b1, w2, b2 = (_arr(a, np.float64) for a in (w1, b1, w2, b2))
        if w1.ndim != 2 or w1.shape[0] != inn:
            raise ValueError(f"score: token dim {inn} != router input dim {w1.shape[0] if w1.ndim else 0}")
        if w2.ndim != 2 or w2.shape[1] != sb.size - 1:
            raise ValueError(f"forward_elastic: router emits {w2.shape[-1]} scores for {sb.size - 1} routed slices")
        d = LayerDesc(out=out, in_=inn, group_size=gs, n_slices=sb.size, slice_bits=_ptr(sb, _i32),
                      scale=_ptr(scale, _f64), zero=_ptr(zero, _f64),
                      codes=(C.cast(C.c_void_p(codes.data_ptr()), C.POINTER(C.c_uint8)) if dev_codes
                             else _ptr(codes, C.c_uint8)),
                      planes=_ptr(planes, C.c_uint64), plane_bits=plane_bits, words_per_row=wpr,
                      router_hidden=w1.shape[1], w1=_ptr(w1, _f64), b1=_ptr(b1, _f64), w2=_ptr(w2, _f64),
                      b2=_ptr(b2, _f64))
        h = C.c_void_p()
        if rows is not None:
            check(lib().mobi_layer_create_rows(C.byref(d), rows[0], rows[1], device, C.byref(h)))
            return cls(h.value, sb.tolist(), rows[1] - rows[0], inn, w1.shape[1], device)
        create = lib().mobi_layer_create_device if dev_codes else lib().mobi_layer_create
        check(create(C.byref(d), device, C.byref(h)))
        return cls(h.value, sb.tolist(), out, inn, w1.shape[1], device)

    def close(self):
        if self._h and self._h.value:
            lib().mobi_layer_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------- queries ----------------
    def reserve(self, max_tokens: int):
        check(lib().mobi_layer_reserve(self._h, max_tokens))

    def device_bytes(self) -> int:
        b = _i64()
        check(lib().mobi_layer_info(self._h, None, None, None, None, C.byref(b)))
        return b.value

    def last_launches(self) -> int:
        n = _i32()
        check(lib().mobi_layer_last_launches(self._h, C.byref(n)))
        return n.value

    KERNEL_IDS = {0: None, 1: "router_dec", 2: "router_tc", 3: "router_tc_cluster", 4: "router_tc_splitk",
                  5: "router_pair128", 6: "router_pair256", 7: "router_simt", 11: "decode_planes",
                  12: "decode_merged", 13: "gemm_splitk", 14: "gemm_pair", 15: "gemm_simt", 16: "gemm_generic"}

    def last_plan(self) -> dict:
        """Kernels the last call on this layer ran (mobi_layer_last_plan): router / GEMM kernel names,
        GEMM grid, launches, token tiles, 256-row weight-tile pairs and GEMM units (tiles x pairs)."""
        a = (_i32 * 8)()
        check(lib().mobi_layer_last_plan(self._h, a))
        return {"router": self.KERNEL_IDS.get(a[0], a[0]), "gemm": self.KERNEL_IDS.get(a[1], a[1]),
                "gemm_ctas": a[2], "launches": a[3], "token_tiles": a[4], "row_pairs": a[5], "units": a[6],
                "tokens": a[7]}

    def set_debug_impl(self, impl: int) -> None:
        """Test hook (per layer): 1 = CUDA-core reference GEMM/router, 0 = production kernels."""
        check(lib().mobi_layer_debug_impl(self._h, impl))

    KERNELS = ("router", "bucket", "gather", "gemm")

    def profile(self, enable: bool = True):
        """Start (or stop) per-kernel CUDA-event timing on the launch stream."""
        check(lib().mobi_layer_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        """{kernel: (total_ms, launches)} accumulated since profile(True)."""
        ms = np.zeros(4, np.float64)
        n = np.zeros(4, np.int64)
        check(lib().mobi_layer_profile_read(self._h, ms.ctypes.data, n.ctypes.data))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(self.KERNELS)}

    def export_router(self):
        w1 = np.zeros((self.inn, self.hidden), np.float32)
        b1 = np.zeros(self.hidden, np.float32)
        w2 = np.zeros((self.hidden, self.n_routed), np.float32)
        b2 = np.zeros(self.n_routed, np.float32)
        check(lib().mobi_layer_export_router(self._h, w1.ctypes.data, b1.ctypes.data, w2.ctypes.data, b2.ctypes.data))
        return w1, b1, w2, b2

    def unpack_codes(self) -> np.ndarray:
        codes = np.zeros((len(self.slice_bits), self.out, self.inn), np.uint8)
        check(lib().mobi_layer_unpack_codes(self._h, codes.ctypes.data))
        return codes

    # ---------------- hot path ----------------
    def _x(self, x: torch.Tensor) -> torch.Tensor:
        if x.dim() != 2 or x.shape[1] != self.inn:
            raise ValueError(f"score: token dim {x.shape[-1]} != router input dim {self.inn}")
        if x.dtype != torch.bfloat16 or not x.is_cuda:
            raise ValueError("MobiLayer expects a CUDA bfloat16 [T, in] tensor")
        return x.contiguous()

    def score(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """router.hpp:63-76: S[T, E-1] fp32."""
        x = self._x(x)
        s = torch.empty((x.shape[0], self.n_routed), dtype=torch.float32, device=x.device)
        check(lib().mobi_score(self._h, x.data_ptr(), x.shape[0], s.data_ptr(), _stream_ptr(stream)))
        return s

    def route(self, x: torch.Tensor, delta: float, stream=None):
        """score -> gate_hard(delta) -> masks -> permute_by_slice. Returns (scores, masks, perm, inverse, counts)."""
        x = self._x(x)
        T = x.shape[0]
        dev = x.device
        s = torch.empty((T, self.n_routed), dtype=torch.float32, device=dev)
        m = torch.empty(T, dtype=torch.uint8, device=dev)
        perm = torch.empty(T, dtype=torch.int32, device=dev)
        inv = torch.empty(T, dtype=torch.int32, device=dev)
        cnt = torch.zeros(1 << len(self.slice_bits), dtype=torch.int32, device=dev)  # bucket_count[m], m < 2^E
        check(lib().mobi_route(self._h, x.data_ptr(), T, float(delta), s.data_ptr(), m.data_ptr(), perm.data_ptr(),
                               inv.data_ptr(), cnt.data_ptr(), _stream_ptr(stream)))
        return s, m, perm, inv, cnt

    def forward(self, x: torch.Tensor, delta: float, y: Optional[torch.Tensor] = None, return_masks: bool = False,
                stream=None):
        """score -> gate_hard(delta) -> forward_elastic(kHard): Y [T, out] bf16."""
        x = self._x(x)
        T = x.shape[0]
        if y is None:
            y = torch.empty((T, self.out), dtype=torch.bfloat16, device=x.device)
        m = torch.empty(T, dtype=torch.uint8, device=x.device) if return_masks else None
        check(lib().mobi_forward(self._h, x.data_ptr(), T, float(delta), y.data_ptr(),
                                 m.data_ptr() if m is not None else None, _stream_ptr(stream)))
        return (y, m) if return_masks else y

    def forward_out(self, x: torch.Tensor, delta: float, dsts: Sequence[int], ldy: int, col0: int = 0,
                    return_masks: bool = False, stream=None):
        """Forward with output placement (mobi_forward_out): Y row t goes to every destination pointer in
        ``dsts`` (device addresses, local or peer-mapped) at ``t*ldy + col0`` -- the fused all-gather of a
        column-parallel shard when ``dsts`` are the full outputs of every rank."""
        x = self._x(x)
        T = x.shape[0]
        if not 1 <= len(dsts) <= 8:
            raise ValueError(f"mobi_out_desc: n_dst {len(dsts)} outside [1,8]")
        d = OutDesc(n_dst=len(dsts), ldy=ldy, col0=col0)
        for k, ptr in enumerate(dsts):
            d.dst[k] = int(ptr)
        m = torch.empty(T, dtype=torch.uint8, device=x.device) if return_masks else None
        check(lib().mobi_forward_out(self._h, x.data_ptr(), T, float(delta), C.byref(d),
                                     m.data_ptr() if m is not None else None, _stream_ptr(stream)))
        return m

    def forward_masked(self, x: torch.Tensor, masks: torch.Tensor, y: Optional[torch.Tensor] = None, stream=None):
        """router.hpp:105-132 forward_elastic with per-token slice masks (bit e-1 <-> slice e)."""
        x = self._x(x)
        T = x.shape[0]
        if masks.numel() != T:
            raise ValueError(f"forward_elastic: gate shape {masks.numel()}x{self.n_routed} != {T}x{self.n_routed}")
        masks = masks.to(device=x.device, dtype=torch.uint8).contiguous()
        if y is None:
            y = torch.empty((T, self.out), dtype=torch.bfloat16, device=x.device)
        check(lib().mobi_forward_masked(self._h, x.data_ptr(), T, masks.data_ptr(), y.data_ptr(),
                                        _stream_ptr(stream)))
        return y

    def forward_gates(self, x: torch.Tensor, gates) -> torch.Tensor:
        """Exactly the reference signature's gate matrix G [T, E-1] (hard: must be binary)."""
        g = torch.as_tensor(np.asarray(gates, dtype=np.float64))
        if g.shape != (x.shape[0], self.n_routed):
            raise ValueError(f"forward_elastic: gate shape {g.shape[0]}x{g.shape[1] if g.dim() > 1 else 0} != "
                             f"{x.shape[0]}x{self.n_routed}")
        if not bool(((g == 0) | (g == 1)).all()):
            raise ValueError("forward_elastic: hard gate not binary")
        masks = torch.ones(x.shape[0], dtype=torch.int64)
        for j in range(self.n_routed):
            masks |= g[:, j].to(torch.int64) << (j + 1)
        return self.forward_masked(x, masks.to(torch.uint8).to(x.device))

    def forward_host(self, x_host: torch.Tensor, delta: float, y_host: Optional[torch.Tensor] = None,
                     masks_host: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """End-to-end call with HOST buffers (bf16 CPU tensors, pinned for best bandwidth)."""
        if x_host.dtype != torch.bfloat16 or x_host.is_cuda or x_host.dim() != 2 or x_host.shape[1] != self.inn:
            raise ValueError("forward_host expects a CPU bfloat16 [T, in] tensor")
        x_host = x_host.contiguous()
        T = x_host.shape[0]
        if y_host is None:
            y_host = torch.empty((T, self.out), dtype=torch.bfloat16)
        check(lib().mobi_forward_host(self._h, x_host.data_ptr(), T, float(delta), y_host.data_ptr(),
                                      masks_host.data_ptr() if masks_host is not None else None,
                                      _stream_ptr(stream)))
        return y_host


# ---------------- CUDA IPC (peer destinations of the fused column-parallel all-gather) ----------------
def ipc_export(t: torch.Tensor):
    """(64-byte CUDA IPC handle of the allocation holding ``t``, ``t``'s byte offset in it)."""
    buf = C.create_string_buffer(64)
    off = _i64()
    check(lib().mobi_ipc_export(C.c_void_p(t.data_ptr()), buf, C.byref(off)))
    return buf.raw, off.value


def ipc_open(handle: bytes, device: int) -> int:
    """Map a peer's exported allocation on ``device``; returns the allocation's base address there."""
    ptr = C.c_void_p()
    check(lib().mobi_ipc_open(C.create_string_buffer(handle, 64), device, C.byref(ptr)))
    return ptr.value


def ipc_close(ptr: int) -> None:
    check(lib().mobi_ipc_close(C.c_void_p(ptr)))


# ---------------- stateless reference-signature helpers ----------------
def permute_by_slice(masks: torch.Tensor, stream=None):
    """bitplane.hpp:178-201 (index part): returns (perm, inverse, groups[(mask, run_length)])."""
    masks = masks.to(torch.uint8).contiguous()
    if not masks.is_cuda:
        raise ValueError("permute_by_slice expects CUDA masks")
    T = masks.numel()
    perm = torch.empty(T, dtype=torch.int32, device=masks.device)
    inv = torch.empty(T, dtype=torch.int32, device=masks.device)
    gm = np.zeros(256, np.uint8)
    gl = np.zeros(256, np.int64)
    ng = _i64()
    check(lib().mobi_permute_by_slice(masks.data_ptr(), T, perm.data_ptr(), inv.data_ptr(), gm.ctypes.data,
                                      gl.ctypes.data, C.byref(ng), _stream_ptr(stream)))
    return perm, inv, [(int(gm[i]), int(gl[i])) for i in range(ng.value)]


def calibrate_threshold(scores: torch.Tensor, rho: float, stream=None) -> float:
    """router.hpp:167-174 over device fp32 scores."""
    s = scores.to(torch.float32).contiguous().reshape(-1)
    out = _f64()
    check(lib().mobi_calibrate_threshold(s.data_ptr() if s.numel() else None, s.numel(), float(rho), C.byref(out),
                                         _stream_ptr(stream)))
    return out.value


def decompose(w: torch.Tensor, group_size: int, slice_bits: Sequence[int], gamma: float, stream=None):
    """slicer.hpp:69-113 + qcore.hpp:122-146 on the GPU (bit-exact): w fp64 [out, in] (CUDA)
    -> (codes uint8 [E,out,in], scale fp64 [out*G], zero fp64 [out*G], clamp_counts)."""
    w = w.to(torch.float64).contiguous()
    out, inn = w.shape
    sb = _arr(slice_bits, np.int32)
    G = (inn + group_size - 1) // group_size
    codes = torch.empty((sb.size, out, inn), dtype=torch.uint8, device=w.device)
    scale = torch.empty(out * G, dtype=torch.float64, device=w.device)
    zero = torch.empty(out * G, dtype=torch.float64, device=w.device)
    cc = np.zeros(sb.size, np.int64)
    check(lib().mobi_decompose(w.data_ptr(), out, inn, group_size, sb.ctypes.data, sb.size, float(gamma),
                               codes.data_ptr(), scale.data_ptr(), zero.data_ptr(), cc.ctypes.data,
                               _stream_ptr(stream)))
    return codes, scale, zero, cc



class BudgetSchedule(C.Structure):
    """trainer::BudgetSchedule (trainer.hpp:45-51); shape 0 log / 1 linear / 2 cosine / 3 exp."""
    _fields_ = [("b_init", C.c_double), ("b_target", C.c_double), ("total_steps", C.c_int64),
                ("shape", C.c_int32), ("reg_weight", C.c_double)]


class _JointScalars(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("data_term", "reg_term", "avg_bits", "sched_b", "loss", "tau")]


_SHAPES = {"log": 0, "logarithmic": 0, "linear": 1, "cosine": 2, "exp": 3, "exponential": 3}


def joint_step(w: torch.Tensor, group_size: int, slice_bits: Sequence[int], gamma_lo, gamma_hi,
               w1: Optional[torch.Tensor], b1, w2, b2, x: torch.Tensor, y_fp: torch.Tensor, sched, t: int,
               force_gates_on: bool = False, backward: bool = True, stream=None) -> dict:
    """One stage-2 calibration step on the GPU (fp64): trainer::joint_forward (trainer.hpp:203-263)
    and, with backward=True, trainer::joint_backward (trainer.hpp:341-396).

    w [out, in], x [T, in], y_fp [T, out] and the router (w1 [in, h], b1 [h], w2 [h, E-1], b2 [E-1]) are
    CUDA fp64 tensors; gamma_lo / gamma_hi are the per-group clip parameters (host arrays,
    out*ceil(in/group_size)); sched = (b_init, b_target, total_steps, shape, reg_weight) with shape an
    int or "log" / "linear" / "cosine" / "exp".  Returns the JointForward scalars, y_hat and (backward)
    d_gamma_lo / d_gamma_hi (numpy) and d_w1 / d_b1 / d_w2 / d_b2 (CUDA tensors).
    """
    dev = x.device
    f64 = lambda a: a.to(device=dev, dtype=torch.float64).contiguous()  # noqa: E731
    w, x, y_fp = f64(w), f64(x), f64(y_fp)
    out, inn = w.shape
    T = x.shape[0]
    sb = _arr(slice_bits, np.int32)
    nr = sb.size - 1
    G = (inn + group_size - 1) // group_size
    glo = _arr(np.broadcast_to(np.asarray(gamma_lo, np.float64), (out * G,)), np.float64)
    ghi = _arr(np.broadcast_to(np.asarray(gamma_hi, np.float64), (out * G,)), np.float64)
    if w1 is None:
        w1 = torch.zeros((inn, 1), dtype=torch.float64, device=dev)
        b1 = torch.zeros(1, dtype=torch.float64, device=dev)
        w2 = torch.zeros((1, max(nr, 1)), dtype=torch.float64, device=dev)
        b2 = torch.zeros(max(nr, 1), dtype=torch.float64, device=dev)
    w1, b1, w2, b2 = f64(w1), f64(b1), f64(w2), f64(b2)
    h = w1.shape[1]
    bi, bt, L, shape, rw = sched
    sc = BudgetSchedule(float(bi), float(bt), int(L), int(_SHAPES.get(shape, shape)), float(rw))
    res = _JointScalars()
    y_hat = torch.empty((T, out), dtype=torch.float64, device=dev)
    g = {}
    if backward:
        g = dict(d_gamma_lo=np.zeros(out * G), d_gamma_hi=np.zeros(out * G), d_w1=torch.empty_like(w1),
                 d_b1=torch.empty_like(b1), d_w2=torch.empty_like(w2), d_b2=torch.empty_like(b2))
    gp = (lambda k: g[k].ctypes.data if isinstance(g[k], np.ndarray) else g[k].data_ptr()) if backward \
        else (lambda k: None)
    with torch.cuda.device(dev):
        check(lib().mobi_joint_step(w.data_ptr(), out, inn, group_size, sb.ctypes.data, sb.size, glo.ctypes.data,
                                    ghi.ctypes.data, w1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr(), h,
                                    x.data_ptr(), y_fp.data_ptr(), T, C.byref(sc), int(t), int(bool(force_gates_on)),
                                    y_hat.data_ptr(), C.byref(res), gp("d_gamma_lo"), gp("d_gamma_hi"), gp("d_w1"),
                                    gp("d_b1"), gp("d_w2"), gp("d_b2"), _stream_ptr(stream)))
    r = {k: getattr(res, k) for k, _ in _JointScalars._fields_}
    r["y_hat"] = y_hat
    r.update(g)
    return r


def msb_step(w: torch.Tensor, group_size: int, msb_bits: int, gamma_lo, gamma_hi, x: torch.Tensor,
             y_fp: torch.Tensor, backward: bool = True, stream=None) -> dict:
    """The stage-1 calibration step on the GPU (fp64): trainer::msb_forward + msb_backward
    (trainer.hpp:404-426) -- slice 1 alone, y_msb = X·W_1ᵀ, loss = MSE and the clip gradients."""
    dev = x.device
    f64 = lambda a: a.to(device=dev, dtype=torch.float64).contiguous()  # noqa: E731
    w, x, y_fp = f64(w), f64(x), f64(y_fp)
    out, inn = w.shape
    G = (inn + group_size - 1) // group_size
    glo = _arr(np.broadcast_to(np.asarray(gamma_lo, np.float64), (out * G,)), np.float64)
    ghi = _arr(np.broadcast_to(np.asarray(gamma_hi, np.float64), (out * G,)), np.float64)
    y = torch.empty((x.shape[0], out), dtype=torch.float64, device=dev)
    loss = C.c_double()
    dlo, dhi = np.zeros(out * G), np.zeros(out * G)
    with torch.cuda.device(dev):
        check(lib().mobi_msb_step(w.data_ptr(), out, inn, group_size, int(msb_bits), glo.ctypes.data, ghi.ctypes.data,
                                  x.data_ptr(), y_fp.data_ptr(), x.shape[0], y.data_ptr(), C.byref(loss),
                                  dlo.ctypes.data if backward else None, dhi.ctypes.data if backward else None,
                                  _stream_ptr(stream)))
    r = dict(y_msb=y, loss=loss.value)
    if backward:
        r.update(d_gamma_lo=dlo, d_gamma_hi=dhi)
    return r


def share_activations(layers: Sequence["MobiLayer"]) -> None:
    """mobi_layers_share_activations: layers that run one after another on one stream (a model stack)
    share one permuted-activation buffer instead of one each.  Reserve every layer first."""
    arr = (C.c_void_p * len(layers))(*[ly._h.value for ly in layers])
    check(lib().mobi_layers_share_activations(arr, len(layers)))
