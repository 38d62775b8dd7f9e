"""MOBI v1 checkpoint ingest.

Reads and writes the reference's binary container bit-exactly
(reference: proj/include/mobi/bench/checkpoint.hpp:15-20 layout, 181-303 section
payloads, 307-388 save/load).  A layer's slice payload stays in the reference's
on-disk form -- the merged code ``INT = c1<<6 | c2<<4 | c3<<2 | c4`` stored as
``bits`` bit-planes, MSB plane first, 64-bit words LSB-first along the input
dim (bitplane.hpp:21-36, 48-73) -- and is handed unchanged to the C-ABI
(``mobi_layer_desc.planes``), which repacks it on the device.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field
from typing import List

import numpy as np

MAGIC = b"MOBI"
VERSION = 1


class CheckpointError(RuntimeError):
    """Mirrors mobi::bench::CheckpointError (checkpoint.hpp:23-25)."""

    def __init__(self, msg: str):
        super().__init__("checkpoint: " + msg)


class _Reader:
    def __init__(self, buf: bytes):
        self.b = buf
        self.p = 0

    def need(self, n):
        if self.p + n > len(self.b):
            raise CheckpointError("section truncated")

    def u8(self):
        self.need(1)
        v = self.b[self.p]
        self.p += 1
        return v

    def u32(self):
        self.need(4)
        v = struct.unpack_from("<I", self.b, self.p)[0]
        self.p += 4
        return v

    def u64(self):
        self.need(8)
        v = struct.unpack_from("<Q", self.b, self.p)[0]
        self.p += 8
        return v

    def f64(self):
        self.need(8)
        v = struct.unpack_from("<d", self.b, self.p)[0]
        self.p += 8
        return v

    def vec_f64(self):
        n = self.u64()
        self.need(8 * n)
        v = np.frombuffer(self.b, "<f8", n, self.p).copy()
        self.p += 8 * n
        return v

    def vec_u64(self):
        n = self.u64()
        self.need(8 * n)
        v = np.frombuffer(self.b, "<u8", n, self.p).copy()
        self.p += 8 * n
        return v

    def vec_i32(self):
        n = self.u64()
        return [struct.unpack("<i", struct.pack("<I", self.u32()))[0] for _ in range(n)]


class _Writer:
    def __init__(self):
        self.parts: List[bytes] = []

    def u8(self, v):
        self.parts.append(struct.pack("<B", v))

    def u32(self, v):
        self.parts.append(struct.pack("<I", v & 0xFFFFFFFF))

    def u64(self, v):
        self.parts.append(struct.pack("<Q", v))

    def f64(self, v):
        self.parts.append(struct.pack("<d", v))

    def vec_f64(self, v):
        v = np.ascontiguousarray(v, "<f8")
        self.u64(v.size)
        self.parts.append(v.tobytes())

    def vec_u64(self, v):
        v = np.ascontiguousarray(v, "<u8")
        self.u64(v.size)
        self.parts.append(v.tobytes())

    def vec_i32(self, v):
        self.u64(len(v))
        for x in v:
            self.u32(x)

    def bytes(self):
        return b"".join(self.parts)


# checkpoint.hpp:181-237 GLOBAL section field order (RunConfig echo).
_GLOBAL_FIELDS = [
    ("model_dim", "u64"), ("model_depth", "u64"), ("group_size", "u64"), ("weight_scale", "f64"),
    ("nsamples", "u64"), ("seqlen", "u64"), ("outlier_frac", "f64"), ("outlier_scale", "f64"),
    ("slice_bits", "vec_i32"), ("epochs", "u64"), ("batch_size", "u64"), ("lr_clip", "f64"),
    ("lr_router", "f64"), ("weight_decay", "f64"), ("gamma_init", "f64"),
    ("stage1_warmup_only", "u8"), ("b_init", "f64"), ("b_target", "f64"), ("shape", "u8"),
    ("reg_weight", "f64"), ("target_bits", "vec_f64"), ("target_ratio", "f64"),
    ("top_frac", "f64"), ("seed", "u64"),
]


@dataclass
class LayerRecord:
    """checkpoint.hpp:30-74."""

    rows: int
    cols: int
    group_size: int
    slice_bits: List[int]
    base_scale: np.ndarray
    base_zero: np.ndarray
    gamma_lo: np.ndarray
    gamma_hi: np.ndarray
    w1: np.ndarray            # [d, h]
    b1: np.ndarray            # [h]
    w2: np.ndarray            # [h, n_routed]
    b2: np.ndarray            # [n_routed]
    threshold: float = 0.0
    step: int = 1
    total_steps: int = 1
    planes: np.ndarray = field(default=None)  # uint64 [bits, rows, words_per_row], MSB plane first
    plane_bits: int = 8

    @property
    def words_per_row(self) -> int:
        return int(self.planes.shape[2])

    def merged_codes(self) -> np.ndarray:
        """bitplane.hpp:75-84 unpack: planes -> merged uint8 code per weight."""
        bits, rows, wpr = self.planes.shape
        out = np.zeros((rows, wpr * 64), np.uint32)
        for b in range(bits):  # bit b lives in plane bits-1-b
            words = self.planes[bits - 1 - b]
            bitsarr = np.unpackbits(words.view(np.uint8).reshape(rows, wpr, 8), axis=2, bitorder="little")
            out |= bitsarr.reshape(rows, wpr * 64).astype(np.uint32) << b
        return out[:, : self.cols].astype(np.uint8)

    def stack(self) -> np.ndarray:
        """checkpoint.hpp:54-73: split merged codes back into [E, rows, cols] slice codes."""
        merged = self.merged_codes()
        total = sum(self.slice_bits)
        shift = total
        codes = []
        for b in self.slice_bits:
            shift -= b
            codes.append(((merged >> shift) & ((1 << b) - 1)).astype(np.uint8))
        return np.stack(codes)


@dataclass
class Checkpoint:
    config: dict
    layers: List[LayerRecord]


def _read_layer(r: _Reader) -> LayerRecord:  # checkpoint.hpp:265-303
    rows, cols, gs = r.u64(), r.u64(), r.u64()
    slice_bits = r.vec_i32()
    scale, zero = r.vec_f64(), r.vec_f64()
    glo, ghi = r.vec_f64(), r.vec_f64()
    d, h, nr = r.u64(), r.u64(), r.u64()
    step, total_steps = r.u64(), r.u64()
    threshold = r.f64()
    w1 = r.vec_f64()
    if w1.size != d * h:
        raise CheckpointError("router w1 size mismatch")
    b1 = r.vec_f64()
    w2 = r.vec_f64()
    if w2.size != h * nr:
        raise CheckpointError("router w2 size mismatch")
    b2 = r.vec_f64()
    bits = r.u32()
    out, inn, wpr = r.u64(), r.u64(), r.u64()
    planes = []
    for _ in range(bits):
        p = r.vec_u64()
        if p.size != out * wpr:
            raise CheckpointError("plane size mismatch")
        planes.append(p.reshape(out, wpr))
    return LayerRecord(rows=rows, cols=cols, group_size=gs, slice_bits=slice_bits, base_scale=scale,
                       base_zero=zero, gamma_lo=glo, gamma_hi=ghi, w1=w1.reshape(d, h), b1=b1,
                       w2=w2.reshape(h, nr), b2=b2, threshold=threshold, step=step,
                       total_steps=total_steps,
                       planes=np.stack(planes) if planes else np.zeros((0, out, wpr), np.uint64),
                       plane_bits=bits)


def _write_layer(w: _Writer, l: LayerRecord) -> None:  # checkpoint.hpp:239-263
    w.u64(l.rows)
    w.u64(l.cols)
    w.u64(l.group_size)
    w.vec_i32(l.slice_bits)
    w.vec_f64(l.base_scale)
    w.vec_f64(l.base_zero)
    w.vec_f64(l.gamma_lo)
    w.vec_f64(l.gamma_hi)
    w.u64(l.w1.shape[0])
    w.u64(l.w1.shape[1])
    w.u64(l.w2.shape[1])
    w.u64(l.step)
    w.u64(l.total_steps)
    w.f64(l.threshold)
    w.vec_f64(l.w1.ravel())
    w.vec_f64(l.b1)
    w.vec_f64(l.w2.ravel())
    w.vec_f64(l.b2)
    w.u32(l.plane_bits)
    w.u64(l.planes.shape[1])
    w.u64(l.cols)
    w.u64(l.planes.shape[2])
    for p in l.planes:
        w.vec_u64(p.ravel())


def loads(data: bytes) -> Checkpoint:
    """checkpoint.hpp:345-388 load_checkpoint."""
    if len(data) < 12:
        raise CheckpointError("file too small")
    if data[:4] != MAGIC:
        raise CheckpointError("bad magic")
    head = _Reader(data[4:])
    version = head.u32()
    if version != VERSION:
        raise CheckpointError(f"version mismatch: file has {version}, expected {VERSION}")
    n = head.u32()
    entries = []
    for _ in range(n):
        tag = bytes(head.u8() for _ in range(8)).split(b"\0", 1)[0].decode()
        off, ln = head.u64(), head.u64()
        if off + ln > len(data):
            raise CheckpointError(f"section '{tag}' out of bounds")
        entries.append((tag, off, ln))
    config, layers, have_global = {}, [], False
    for tag, off, ln in entries:
        r = _Reader(data[off:off + ln])
        if tag == "GLOBAL":
            for name, kind in _GLOBAL_FIELDS:
                config[name] = getattr(r, kind)()
            have_global = True
        elif tag.startswith("LAYER"):
            layers.append(_read_layer(r))
        else:
            raise CheckpointError(f"unknown section tag '{tag}'")
    if not have_global:
        raise CheckpointError("missing GLOBAL section")
    return Checkpoint(config=config, layers=layers)


def load(path) -> Checkpoint:
    try:
        with open(path, "rb") as f:
            return loads(f.read())
    except OSError:
        raise CheckpointError(f"cannot open {path}")


def dumps(ck: Checkpoint) -> bytes:
    """checkpoint.hpp:307-343 save_checkpoint."""
    sections = []
    g = _Writer()
    for name, kind in _GLOBAL_FIELDS:
        getattr(g, kind)(ck.config[name])
    sections.append(("GLOBAL", g.bytes()))
    for i, l in enumerate(ck.layers):
        w = _Writer()
        _write_layer(w, l)
        sections.append((f"LAYER{i:03d}", w.bytes()))
    hdr = _Writer()
    hdr.u32(VERSION)
    hdr.u32(len(sections))
    off = 4 + 8 + len(sections) * 24
    for tag, body in sections:
        t8 = tag.encode()[:8].ljust(8, b"\0")
        hdr.parts.append(t8)
        hdr.u64(off)
        hdr.u64(len(body))
        off += len(body)
    return MAGIC + hdr.bytes() + b"".join(b for _, b in sections)
