"""numpy front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two back-ends with the same Python surface:
  * ``restatement()`` -- oracle/lib/libmobi_oracle.so, the C restatement of the
    reference hot path (mobi_oracle.c);
  * ``reference()``   -- oracle/_ref/libmobi_ref.so, the UNMODIFIED reference
    headers compiled where they lie (ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_ORACLE = HERE / "lib" / "libmobi_oracle.so"
LIB_REF = HERE / "_ref" / "libmobi_ref.so"

_i64 = C.c_int64
_i32 = C.c_int32
_dbl = C.c_double
_p = C.c_void_p


def build() -> None:
    """Build the oracle libraries (reference part only when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _i32a(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class OracleError(ValueError):
    """Mirrors std::invalid_argument raised by MOBI_CHECK."""


class _Backend:
    def __init__(self, path: Path, prefix: str):
        if not path.exists():
            build()
        self.lib = C.CDLL(str(path))
        self.prefix = prefix
        self.kind = "reference" if prefix == "ref_" else "port"
        getattr(self.lib, prefix + "last_error").restype = C.c_char_p

    def _call(self, name, *args):
        fn = getattr(self.lib, self.prefix + name)
        rc = fn(*args)
        if rc != 0:
            msg = getattr(self.lib, self.prefix + "last_error")().decode()
            if rc == 1:
                raise OracleError(msg)
            raise RuntimeError(msg)

    # ---- router.hpp ----
    def score(self, x, w1, b1, w2, b2):
        x, w1, b1, w2, b2 = map(_f64, (x, w1, b1, w2, b2))
        T, d = x.shape
        h = w1.shape[1]
        nr = w2.shape[1]
        if w1.shape[0] != d:
            raise OracleError(f"score: token dim {d} != router input dim {w1.shape[0]}")
        s = np.zeros((T, nr))
        self._call("score", _ptr(x), _i64(T), _i64(d), _ptr(w1), _ptr(b1), _i64(h), _ptr(w2),
                   _ptr(b2), _i64(nr), _ptr(s))
        return s

    def gate_hard(self, s, delta):
        s = _f64(s)
        g = np.zeros_like(s)
        if self.prefix == "ref_":
            self._call("gate_hard", _ptr(s), _i64(s.shape[0]), _i64(s.shape[1] if s.ndim > 1 else 1),
                       _dbl(delta), _ptr(g))
        else:
            self.lib.orc_gate_hard(_ptr(s), _i64(s.size), _dbl(delta), _ptr(g))
        return g

    def forward_elastic(self, x, codes, slice_bits, scale, zero, group_size, gates, hard=True):
        x, codes, sb = _f64(x), _u8(codes), _i32a(slice_bits)
        scale, zero, gates = _f64(scale), _f64(zero), _f64(gates)
        T, d = x.shape
        E, out, inn = codes.shape
        if gates.shape != (T, E - 1):
            raise OracleError(f"forward_elastic: gate shape {gates.shape[0]}x{gates.shape[1]} != {T}x{E - 1}")
        y = np.zeros((T, out))
        self._call("forward_elastic", _ptr(x), _i64(T), _i64(inn), _ptr(codes), _i32(E), _ptr(sb),
                   _ptr(scale), _ptr(zero), _i64(out), _i64(group_size), _ptr(gates),
                   C.c_int(1 if hard else 0), _ptr(y))
        return y

    def calibrate_threshold(self, scores, rho):
        s = _f64(np.ravel(scores))
        out = _dbl()
        self._call("calibrate_threshold", _ptr(s), _i64(s.size), _dbl(rho), C.byref(out))
        return out.value

    def avg_bits(self, gates, slice_bits):
        g, sb = _f64(gates), _i32a(slice_bits)
        out = _dbl()
        self._call("avg_bits", _ptr(g), _i64(g.shape[0]), _i64(g.shape[1]), _ptr(sb), _i32(sb.size),
                   C.byref(out))
        return out.value

    def ratio_from_target_bits(self, target, slice_bits):
        sb = _i32a(slice_bits)
        out = _dbl()
        self._call("ratio_from_target_bits", _dbl(target), _ptr(sb), _i32(sb.size), C.byref(out))
        return out.value

    # ---- qcore / slicer ----
    def params_from_clip(self, w, group_size, bits, gamma_lo, gamma_hi=None):
        w = _f64(w)
        rows, cols = w.shape
        ng = rows * ((cols + group_size - 1) // group_size)
        glo = _f64(np.broadcast_to(np.asarray(gamma_lo, np.float64), (ng,)))
        ghi = _f64(np.broadcast_to(np.asarray(gamma_lo if gamma_hi is None else gamma_hi, np.float64), (ng,)))
        scale = np.zeros(ng)
        zero = np.zeros(ng)
        self._call("params_from_clip", _ptr(w), _i64(rows), _i64(cols), _i64(group_size), _ptr(glo),
                   _ptr(ghi), C.c_int(bits), _ptr(scale), _ptr(zero))
        return scale, zero

    def decompose(self, w, group_size, scale, zero, slice_bits):
        w, scale, zero, sb = _f64(w), _f64(scale), _f64(zero), _i32a(slice_bits)
        rows, cols = w.shape
        codes = np.zeros((sb.size, rows, cols), np.uint8)
        cmask = np.zeros((rows, cols), np.uint8)
        counts = np.zeros(sb.size, np.int64)
        self._call("decompose", _ptr(w), _i64(rows), _i64(cols), _i64(group_size), _ptr(scale),
                   _ptr(zero), _ptr(sb), _i32(sb.size), _ptr(codes), _ptr(cmask), _ptr(counts))
        return codes, cmask, counts

    def reconstruct(self, codes, slice_bits, scale, zero, group_size, k):
        codes, sb, scale, zero = _u8(codes), _i32a(slice_bits), _f64(scale), _f64(zero)
        E, rows, cols = codes.shape
        out = np.zeros((rows, cols))
        self._call("reconstruct", _ptr(codes), _i64(rows), _i64(cols), _i64(group_size), _ptr(sb),
                   _i32(E), _ptr(scale), _ptr(zero), _i32(k), _ptr(out))
        return out

    def merge_codes(self, codes, slice_bits, k=None):
        codes, sb = _u8(codes), _i32a(slice_bits)
        E, rows, cols = codes.shape
        k = E if k is None else k
        merged = np.zeros((rows, cols), np.uint8)
        if self.prefix == "ref_":
            self._call("merge_codes", _ptr(codes), _i64(rows), _i64(cols), _ptr(sb), _i32(E), _i32(k),
                       _ptr(merged))
        else:
            self._call("merge_codes", _ptr(codes), _i64(rows * cols), _ptr(sb), _i32(E), _i32(k),
                       _ptr(merged))
        return merged

    # ---- bitplane ----
    def pack_bit_major(self, codes, bits):
        codes = _u8(codes)
        rows, cols = codes.shape
        wpr = (cols + 63) // 64
        planes = np.zeros((bits, rows, wpr), np.uint64)
        self._call("pack_bit_major", _ptr(codes), _i64(rows), _i64(cols), C.c_int(bits), _ptr(planes))
        return planes

    def layer_stack(self, planes, cols, slice_bits):
        """checkpoint.hpp:54 LayerRecord::stack(): merged planes -> [E, rows, cols] slice codes."""
        planes, sb = np.ascontiguousarray(planes, np.uint64), _i32a(slice_bits)
        bits, rows, wpr = planes.shape
        codes = np.zeros((sb.size, rows, cols), np.uint8)
        if self.prefix == "ref_":
            self._call("layer_stack", _ptr(planes), _i64(rows), _i64(cols), C.c_int(bits), _i64(wpr),
                       _ptr(sb), _i32(sb.size), _ptr(codes))
        else:
            merged = np.zeros((rows, cols), np.uint8)
            self._call("unpack", _ptr(planes), _i64(rows), _i64(cols), C.c_int(bits), _i64(wpr),
                       _ptr(merged))
            self._call("split_merged", _ptr(merged), _i64(rows * cols), _ptr(sb), _i32(sb.size),
                       _ptr(codes))
        return codes

    def bitplane_matmul(self, x, planes, cols, group_size, scale, zero, active):
        x, planes = _f64(x), np.ascontiguousarray(planes, np.uint64)
        scale, zero, act = _f64(scale), _f64(zero), _i32a(active)
        bits, out, wpr = planes.shape
        T = x.shape[0]
        y = np.zeros((T, out))
        self._call("bitplane_matmul", _ptr(x), _i64(T), _ptr(planes), _i64(out), _i64(cols),
                   C.c_int(bits), _i64(wpr), _i64(group_size), _ptr(scale), _ptr(zero), _ptr(act),
                   _i32(act.size), _ptr(y))
        return y

    def permute_by_slice(self, tokens, masks):
        tokens, masks = _f64(tokens), _u8(masks)
        T = tokens.shape[0]
        cols = tokens.shape[1] if tokens.ndim > 1 else 1
        if masks.size != T:
            raise OracleError(f"permute_by_slice: {masks.size} assignments for {T} tokens")
        permuted = np.zeros((T, cols))
        perm = np.zeros(T, np.int64)
        inv = np.zeros(T, np.int64)
        gm = np.zeros(256, np.uint8)
        gl = np.zeros(256, np.int64)
        ng = _i64()
        self._call("permute_by_slice", _ptr(tokens), _i64(T), _i64(cols), _ptr(masks), _ptr(permuted),
                   _ptr(perm), _ptr(inv), _ptr(gm), _ptr(gl), C.byref(ng))
        groups = [(int(gm[i]), int(gl[i])) for i in range(ng.value)]
        return permuted, perm, inv, groups


    # ---- trainer.hpp (stage-2 calibration step; the reference backend only) ----
    def joint_step(self, w, group_size, slice_bits, gamma_lo, gamma_hi, w1, b1, w2, b2, x, y_fp, sched, t,
                   force_gates_on=False, backward=True):
        """trainer.hpp:203-263 joint_forward (+ 341-396 joint_backward).  sched = (b_init, b_target,
        total_steps, shape 0 log / 1 linear / 2 cosine / 3 exp, reg_weight)."""
        w, x, y_fp, w1, b1, w2, b2 = map(_f64, (w, x, y_fp, w1, b1, w2, b2))
        sb = _i32a(slice_bits)
        out, inn = w.shape
        T = x.shape[0]
        h = w1.shape[1]
        ng = out * ((inn + group_size - 1) // group_size)
        glo, ghi = _f64(gamma_lo), _f64(gamma_hi)
        y_hat = np.zeros((T, out))
        sc = np.zeros(6)
        g = dict(d_gamma_lo=np.zeros(ng), d_gamma_hi=np.zeros(ng), d_w1=np.zeros_like(w1), d_b1=np.zeros(h),
                 d_w2=np.zeros_like(w2), d_b2=np.zeros(w2.shape[1]))
        bi, bt, L, shape, rw = sched
        gp = (lambda k: _ptr(g[k])) if backward else (lambda k: None)
        self._call("joint_step", _ptr(w), _i64(out), _i64(inn), _i64(group_size), _ptr(sb), _i32(sb.size),
                   _ptr(glo), _ptr(ghi), _ptr(w1), _ptr(b1), _ptr(w2), _ptr(b2), _i64(h), _ptr(x), _ptr(y_fp),
                   _i64(T), _dbl(bi), _dbl(bt), _i64(L), _i32(shape), _dbl(rw), _i64(t), _i32(int(force_gates_on)),
                   _ptr(y_hat), _ptr(sc), gp("d_gamma_lo"), gp("d_gamma_hi"), gp("d_w1"), gp("d_b1"), gp("d_w2"),
                   gp("d_b2"))
        r = dict(zip(("data_term", "reg_term", "avg_bits", "sched_b", "loss", "tau"), sc.tolist()))
        r["y_hat"] = y_hat
        if backward:
            r.update(g)
        return r

    def msb_step(self, w, group_size, slice_bits, gamma_lo, gamma_hi, x, y_fp):
        """trainer.hpp:404-426 msb_forward + msb_backward."""
        w, x, y_fp, glo, ghi = map(_f64, (w, x, y_fp, gamma_lo, gamma_hi))
        sb = _i32a(slice_bits)
        out, inn = w.shape
        T = x.shape[0]
        ng = out * ((inn + group_size - 1) // group_size)
        y = np.zeros((T, out))
        loss = _dbl()
        dlo, dhi = np.zeros(ng), np.zeros(ng)
        self._call("msb_step", _ptr(w), _i64(out), _i64(inn), _i64(group_size), _ptr(sb), _i32(sb.size), _ptr(glo),
                   _ptr(ghi), _ptr(x), _ptr(y_fp), _i64(T), _ptr(y), C.byref(loss), _ptr(dlo), _ptr(dhi))
        return dict(y_msb=y, loss=loss.value, d_gamma_lo=dlo, d_gamma_hi=dhi)


def restatement() -> _Backend:
    return _Backend(LIB_ORACLE, "orc_")


def reference() -> _Backend:
    return _Backend(LIB_REF, "ref_")


def masks_from_gates(gates) -> np.ndarray:
    """bitplane.hpp:203-206 convention: bit e-1 <-> slice e, slice 1 always on."""
    g = np.asarray(gates) > 0.5
    m = np.ones(g.shape[0], np.uint8)
    for j in range(g.shape[1]):
        m |= (g[:, j].astype(np.uint8) << (j + 1))
    return m


# ---- seeded generators restating the reference's fixture recipes (C restatement back-end) ----
class Rng:
    """common.hpp:140-201 Rng (xoshiro256++), driven through the C restatement."""

    class _S(C.Structure):
        _fields_ = [("s", C.c_uint64 * 4), ("spare", C.c_double), ("has_spare", C.c_int)]

    def __init__(self, seed: int):
        self._lib = restatement().lib
        self._st = Rng._S()
        self._lib.orc_rng_init(C.byref(self._st), C.c_uint64(seed))
        self._lib.orc_rng_next_u64.restype = C.c_uint64
        self._lib.orc_rng_uniform.restype = C.c_double
        self._lib.orc_rng_normal.restype = C.c_double
        self._lib.orc_rng_uniform_index.restype = C.c_uint64

    def normal(self, n=None, scale=1.0):
        if n is None:
            return self._lib.orc_rng_normal(C.byref(self._st))
        out = np.zeros(n)
        self._lib.orc_rng_fill_normal(C.byref(self._st), _ptr(out), _i64(n), _dbl(scale))
        return out

    def uniform(self):
        return self._lib.orc_rng_uniform(C.byref(self._st))

    def uniform_index(self, n):
        return int(self._lib.orc_rng_uniform_index(C.byref(self._st), C.c_uint64(n)))

    def router_init(self, d, n_routed, hidden=0):
        h = hidden if hidden else max(1, d // 4)
        w1, b1 = np.zeros((d, h)), np.zeros(h)
        w2, b2 = np.zeros((h, n_routed)), np.zeros(n_routed)
        self._lib.orc_router_init(_i64(d), _i64(n_routed), _i64(hidden), C.byref(self._st), _ptr(w1),
                                  _ptr(b1), _ptr(w2), _ptr(b2))
        return w1, b1, w2, b2


def gen_calibset(nsamples, seqlen, dim, outlier_frac, outlier_scale, seed):
    lib = restatement().lib
    out = np.zeros((nsamples, seqlen, dim))
    chans = np.zeros(max(1, dim), np.int64)
    n_out = _i64()
    lib.orc_gen_calibset(_i64(nsamples), _i64(seqlen), _i64(dim), _dbl(outlier_frac),
                         _dbl(outlier_scale), C.c_uint64(seed), _ptr(out), _ptr(chans), C.byref(n_out))
    return out, chans[: n_out.value]


def gen_model(dim, depth, seed, weight_scale):
    lib = restatement().lib
    out = np.zeros((depth, dim, dim))
    lib.orc_gen_model(_i64(dim), _i64(depth), C.c_uint64(seed), _dbl(weight_scale), _ptr(out))
    return out


def synthetic_layer(out_dim, in_dim, *, seed=1, group_size=128, slice_bits=(2, 2, 2, 2),
                    weight_sd=0.02, gamma=4.0, hidden=0, w2_sd=0.3, b2_sd=0.1, backend=None):
    """SURVEY 8(d) recipe: W ~ N(0, sd^2) -> params_from_clip(identity_init(gamma)) -> decompose;
    router = RouterState::init(in, E-1, .., h) then w2 <- 0.3 N(0,1), b2 <- 0.1 N(0,1)
    (tools/mobi.cpp:211-212)."""
    be = backend or restatement()
    rng = Rng(seed)
    w = rng.normal(out_dim * in_dim, weight_sd).reshape(out_dim, in_dim)
    scale, zero = be.params_from_clip(w, group_size, slice_bits[0], gamma)
    codes, _, counts = be.decompose(w, group_size, scale, zero, slice_bits)
    w1, b1, w2, b2 = rng.router_init(in_dim, len(slice_bits) - 1, hidden)
    w2 = rng.normal(w2.size, w2_sd).reshape(w2.shape)
    b2 = rng.normal(b2.size, b2_sd)
    return dict(w=w, scale=scale, zero=zero, codes=codes, clamp_counts=counts, slice_bits=list(slice_bits),
                group_size=group_size, w1=w1, b1=b1, w2=w2, b2=b2)


# ---------------------------------------------------------------------------------------------
# Stage-2 calibration step, restated in numpy: trainer.hpp:203-263 joint_forward
# and trainer.hpp:341-396 joint_backward, with the bit-exact C restatement for params_from_clip /
# decompose (qcore.hpp:122-146, slicer.hpp:69-113).  Matrix products use numpy's summation order,
# so this is pinned to the reference within fp64 rounding (tests/test_oracle.py), not bit-for-bit.
# ---------------------------------------------------------------------------------------------

def _sigmoid(v):
    v = np.asarray(v, np.float64)
    e = np.exp(-np.abs(v))
    return np.where(v >= 0.0, 1.0 / (1.0 + e), e / (1.0 + e))  # common.hpp:125-131


def schedule_value(sched, t):
    """trainer.hpp:52-73."""
    bi, bt, L, shape, _ = sched
    if not 1 <= t <= L:
        raise OracleError(f"schedule_value: step {t} outside [1,{L}]")
    frac = t / L
    if shape == 0:
        return bt if t == L else bi - (bi - bt) * np.log(t) / np.log(L)
    if shape == 1:
        return bi - (bi - bt) * frac
    if shape == 2:
        return bt + (bi - bt) * (1.0 + np.cos(np.pi * frac)) / 2.0
    return bi * (bt / bi) ** frac


def group_stats(w, group_size):
    """qcore.hpp:75-111 GroupStats::from_weights: per (row, group) min, max, ref = clamp(0, min, max)."""
    out, inn = w.shape
    G = (inn + group_size - 1) // group_size
    pad = np.full((out, G * group_size), np.nan)
    pad[:, :inn] = w
    blk = pad.reshape(out, G, group_size)
    mn = np.nanmin(blk, axis=2).reshape(-1)
    mx = np.nanmax(blk, axis=2).reshape(-1)
    ref = np.minimum(np.maximum(0.0, mn), mx)
    return mn, mx, ref


def joint_step_np(w, group_size, slice_bits, gamma_lo, gamma_hi, w1, b1, w2, b2, x, y_fp, sched, t,
                  force_gates_on=False, backward=True, slice1_only=False):
    orc = restatement()
    w, x, y_fp = _f64(w), _f64(x), _f64(y_fp)
    sb = [int(b) for b in slice_bits]
    E, nr = len(sb), len(sb) - 1
    out, inn = w.shape
    T = x.shape[0]
    G = (inn + group_size - 1) // group_size
    glo, ghi = _f64(gamma_lo), _f64(gamma_hi)
    scale, zero = orc.params_from_clip(w, group_size, sb[0], glo, ghi)
    codes, _, _ = orc.decompose(w, group_size, scale, zero, sb)
    if slice1_only:  # msb_forward: slice 1 alone
        sb, E, nr, codes = sb[:1], 1, 0, codes[:1]
    gidx = (np.arange(out)[:, None] * G + np.arange(inn)[None, :] // group_size)
    P, frames = [], []
    before = 0
    for e in range(1, E + 1):
        unit = np.ldexp(1.0, -before)
        mid = 0.0 if e == 1 else np.ldexp(1.0, sb[e - 1] - 1)
        s_e = scale[gidx] * unit
        z_e = zero[gidx] if e == 1 else mid
        We = s_e * (codes[e - 1].astype(np.float64) - z_e + 0.5)  # qcore.hpp:180-197 with slice_params(e)
        P.append(x @ We.T)
        frames.append((codes[e - 1].astype(np.float64) - mid + 0.5) * unit)
        before += sb[e - 1]
    L = sched[2]
    hard = False
    tau = 0.0
    if force_gates_on:
        gates = np.ones((T, nr))
        hpre = hact = np.zeros((T, w1.shape[1]))
        hard = True
    else:
        hpre = x @ _f64(w1) + _f64(b1)[None, :]
        hact = hpre * _sigmoid(hpre)
        scores = hact @ _f64(w2) + _f64(b2)[None, :]
        hard = t == L
        if hard:
            gates = (scores > 0.0).astype(np.float64)
        else:
            ll = np.log(L)
            tau = ll / (ll - np.log(t))
            gates = _sigmoid(tau * scores)
    y_hat = P[0].copy()
    for e in range(2, E + 1):
        y_hat += gates[:, e - 2:e - 1] * P[e - 1]
    data_term = float(np.mean((y_hat - y_fp) ** 2))
    bits = sb[0] + ((gates > 0.5) * np.asarray(sb[1:], np.float64)[None, :]).sum(axis=1)
    avg_bits = float(bits.mean())
    sched_b = float(schedule_value(sched, t))
    reg_term = (avg_bits - sched_b) * float(gates.sum())
    r = dict(data_term=data_term, reg_term=reg_term, avg_bits=avg_bits, sched_b=sched_b,
             loss=data_term + sched[4] * reg_term, tau=tau, y_hat=y_hat)
    if not backward:
        return r
    resid = 2.0 / y_hat.size * (y_hat - y_fp)
    qmax1 = float((1 << sb[0]) - 1)
    d_lo = np.zeros(out * G)
    d_hi = np.zeros(out * G)
    d1 = None
    for e in range(1, E + 1):
        dm = resid.T @ x if e == 1 else (resid * gates[:, e - 2:e - 1]).T @ x
        if e == 1:
            d1 = dm
        fr = dm * frames[e - 1] / qmax1
        np.add.at(d_hi, gidx, fr)
        np.add.at(d_lo, gidx, (dm - fr) if e == 1 else -fr)
    mn, mx, ref = group_stats(w, group_size)
    lo = ref + _sigmoid(glo) * (mn - ref)
    hi = ref + _sigmoid(ghi) * (mx - ref)
    floored = ~((hi - lo) / qmax1 > 1e-8)
    sg_lo = _sigmoid(glo) * (1.0 - _sigmoid(glo))
    sg_hi = _sigmoid(ghi) * (1.0 - _sigmoid(ghi))
    dg_lo = d_lo * sg_lo * (mn - ref)
    dg_hi = np.where(floored, 0.0, d_hi * sg_hi * (mx - ref))
    if floored.any():
        s1 = np.zeros(out * G)
        np.add.at(s1, gidx, d1)
        dg_lo = np.where(floored, s1 * sg_lo * (mn - ref), dg_lo)
    r.update(d_gamma_lo=dg_lo, d_gamma_hi=dg_hi)
    h = _f64(w1).shape[1]
    if hard:
        r.update(d_w1=np.zeros_like(_f64(w1)), d_b1=np.zeros(h), d_w2=np.zeros_like(_f64(w2)), d_b2=np.zeros(nr))
        return r
    reg_coeff = sched[4] * (avg_bits - sched_b)
    d_gate = np.stack([(resid * P[e + 1]).sum(axis=1) for e in range(nr)], axis=1) + reg_coeff
    d_score = d_gate * tau * gates * (1.0 - gates)
    d_act = (d_score @ _f64(w2).T) * (_sigmoid(hpre) * (1.0 + hpre * (1.0 - _sigmoid(hpre))))
    r.update(d_w2=hact.T @ d_score, d_b2=d_score.sum(axis=0), d_w1=x.T @ d_act, d_b1=d_act.sum(axis=0))
    return r


def msb_step_np(w, group_size, slice_bits, gamma_lo, gamma_hi, x, y_fp):
    """trainer.hpp:404-426: the stage-1 step is the joint step's slice-1 part (quantize_floor with the
    clip's base params is decompose's first slice), without router or regulariser."""
    r = joint_step_np(w, group_size, [slice_bits[0], 1], gamma_lo, gamma_hi, np.zeros((w.shape[1], 1)), np.zeros(1),
                      np.zeros((1, 1)), np.zeros(1), x, y_fp, (0.0, 0.0, 1, 0, 0.0), 1, force_gates_on=True,
                      slice1_only=True)
    return dict(y_msb=r["y_hat"], loss=r["data_term"], d_gamma_lo=r["d_gamma_lo"], d_gamma_hi=r["d_gamma_hi"])
