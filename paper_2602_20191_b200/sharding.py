"""Multi-GPU partitioning of the MoBi linear layer.

The layer shards two ways, both exact:

* column-parallel (split ``out``): rank p owns the weight rows [r0_p, r1_p) of every slice plus those
  rows' group parameters -- groups never span rows (qcore.hpp:19-34, ``g = r*ceil(in/gs) + c/gs``), so
  the split is exact.  The router depends only on X, so it is replicated: every rank computes the
  same scores and masks (router.hpp:63-103) and runs route -> bucket -> GEMM on its rows.  The one
  exchange step is an all-gather of the [T, rows_p] outputs over NVLink (NCCL), re-interleaved to
  [T, out].
* token-sharded (split ``T``): replicated layers, rank p forwards tokens [t0_p, t1_p); tokens are
  independent (router.hpp:105-132), so there is no data-path collective.

One process per GPU; ``torch.distributed`` is the plumbing.  The row slicing and the re-interleave
are host logic and are tested on CPU with ``gloo`` (tests/test_sharding.py); the per-rank forward
is the single-GPU C-ABI path.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch


def balanced_ranges(n: int, world: int, align: int = 1):
    """Contiguous [lo, hi) ranges covering [0, n): equal sizes rounded up to ``align`` (the last may be
    shorter or empty)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    per = -(-n // world)
    per = -(-per // align) * align
    return [(min(n, p * per), min(n, (p + 1) * per)) for p in range(world)], per


def shard_stack_rows(codes: np.ndarray, scale: np.ndarray, zero: np.ndarray, group_size: int, r0: int, r1: int):
    """Rows [r0, r1) of a SliceStack: codes [E, out, in] and the per-group base params
    scale/zero [out * ceil(in/gs)] (row-major groups, qcore.hpp:30-34)."""
    E, out, inn = codes.shape
    G = -(-inn // group_size)
    if not (0 <= r0 <= r1 <= out):
        raise ValueError(f"shard rows [{r0},{r1}) outside [0,{out})")
    sc = np.asarray(scale).reshape(out, G)[r0:r1].reshape(-1)
    ze = np.asarray(zero).reshape(out, G)[r0:r1].reshape(-1)
    return np.ascontiguousarray(codes[:, r0:r1, :]), np.ascontiguousarray(sc), np.ascontiguousarray(ze)


def interleave_columns(gathered: torch.Tensor, world: int, T: int, per: int, out: int) -> torch.Tensor:
    """All-gather result [world * T, per] (rank-major) -> [T, out]."""
    return gathered.view(world, T, per).permute(1, 0, 2).reshape(T, world * per)[:, :out]


def all_gather_columns(y_local: torch.Tensor, per: int, out: int, group=None) -> torch.Tensor:
    """[T, rows_p] on every rank -> [T, out] on every rank (one NCCL all-gather over NVLink)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    T = y_local.shape[0]
    if y_local.shape[1] != per:  # the last rank's shard may be short: pad to the common width
        pad = torch.zeros((T, per), dtype=y_local.dtype, device=y_local.device)
        pad[:, : y_local.shape[1]] = y_local
        y_local = pad
    gathered = torch.empty((world * T, per), dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(gathered, y_local.contiguous(), group=group)
    return interleave_columns(gathered, world, T, per, out)


class ColumnParallelMobiLayer:
    """A MobiLayer whose weight rows are split across the ranks of ``group`` (column-parallel linear).

    Built from the full SliceStack + RouterState (the reference's objects); every rank keeps the full
    router and its own rows.  ``forward`` returns the full [T, out] output on every rank.  Collectives:

    * ``"peer"`` (fused): every rank owns a full [T, out] output buffer mapped into every other rank
      (CUDA IPC over NVLink); the GEMM epilogue stores each finished tile into all of them at this
      rank's column offset (mobi_forward_out), so the all-gather overlaps the compute tile by tile and
      needs no re-interleave.  A one-element all-reduce after the GEMM orders the peers' reads.
    * ``"nccl"``: the epilogue writes this rank's [T, rows] block straight into its slot of a
      rank-major [P][T][per] buffer, one in-place NCCL all-gather fills the others, one copy pass
      interleaves into [T, out].
    * ``"auto"`` (default): ``"peer"`` when the ranks are on distinct devices and the IPC mapping
      works and its first output equals the NCCL path's, else ``"nccl"``.
    """

    def __init__(self, codes, slice_bits: Sequence[int], scale, zero, group_size: int, w1, b1, w2, b2,
                 device: int, rank: int, world: int, group=None, row_align: int = 128, collective: str = "auto"):
        from .layer import MobiLayer
        codes = np.asarray(codes, np.uint8)
        self.out = codes.shape[1]
        self.inn = codes.shape[2]
        ranges, self.per = balanced_ranges(self.out, world, row_align)
        self.r0, self.r1 = ranges[rank]
        if self.r1 <= self.r0:
            raise ValueError(f"column-parallel: rank {rank} of {world} owns no rows of {self.out}")
        self.local = MobiLayer.from_stack_rows(codes, slice_bits, scale, zero, group_size, w1, b1, w2, b2,
                                               self.r0, self.r1, device=device)
        self.rank, self.world, self.group, self.device = rank, world, group, device
        self.want = collective
        self.collective = "nccl"
        self._T = 0
        self._bufs = None     # peer mode: [2] double-buffered full outputs [T, out] of this rank
        self._peers = None    # peer mode: [2][world] destination addresses
        self._opened = []
        self._gbuf = None     # nccl mode: rank-major [world, T, per]
        self._flip = 0

    # ---- buffers ----
    def reserve(self, max_tokens: int):
        self.local.reserve(max_tokens)
        self._setup(max_tokens)

    def _setup(self, T: int):
        if T <= self._T:
            return
        import torch.distributed as dist
        dev = torch.device("cuda", self.device)
        self._close_peers()
        self._T = T
        self._gbuf = torch.zeros((self.world, T, self.per), dtype=torch.bfloat16, device=dev)
        if self.want == "nccl" or self.world == 1:
            self.collective = "nccl" if self.world > 1 else "none"
            return
        try:
            from .layer import ipc_export, ipc_open
            self._bufs = [torch.zeros((T, self.out), dtype=torch.bfloat16, device=dev) for _ in range(2)]
            mine = [ipc_export(b) for b in self._bufs]
            devs = [None] * self.world
            props = torch.cuda.get_device_properties(dev)
            ident = str(getattr(props, "uuid", self.device))
            dist.all_gather_object(devs, (ident, mine), group=self.group)
            uuids = [d[0] for d in devs]
            if len(set(uuids)) != self.world and self.want == "auto":
                raise RuntimeError("ranks share a device")
            peers = [[0] * self.world for _ in range(2)]
            for q, (_, handles) in enumerate(devs):
                for k in range(2):
                    if q == self.rank:
                        peers[k][q] = self._bufs[k].data_ptr()
                    else:
                        base = ipc_open(handles[k][0], self.device)
                        self._opened.append(base)
                        peers[k][q] = base + handles[k][1]
            self._peers = peers
            self.collective = "peer"
        except Exception:
            if self.want == "peer":
                raise
            self._close_peers()
            self.collective = "nccl"

    def _close_peers(self):
        if self._opened:
            from .layer import ipc_close
            torch.cuda.synchronize(self.device)
            for b in self._opened:
                try:
                    ipc_close(b)
                except Exception:
                    pass
        self._opened = []
        self._peers = None
        self._bufs = None

    def __del__(self):
        try:
            self._close_peers()
        except Exception:
            pass

    # ---- forward ----
    def forward(self, x: torch.Tensor, delta: float, y: Optional[torch.Tensor] = None, return_masks: bool = False):
        """Full [T, out] output on every rank (into ``y`` when given; in peer mode the returned tensor is
        one of two internal buffers, valid until the second-next call)."""
        import torch.distributed as dist
        T = x.shape[0]
        self._setup(T)
        if self.collective == "peer":
            k = self._flip
            self._flip ^= 1
            m = self.local.forward_out(x, delta, self._peers[k], ldy=self.out, col0=self.r0, return_masks=return_masks)
            # every rank's epilogue has stored into this rank's buffer once all reached this point
            flag = torch.ones(1, dtype=torch.float32, device=x.device)
            dist.all_reduce(flag, group=self.group)
            full = self._bufs[k][:T]
            if y is not None:
                y.copy_(full)
                full = y
        else:
            g = self._gbuf[:, :T] if T == self._T else torch.empty((self.world, T, self.per), dtype=torch.bfloat16,
                                                                     device=x.device)
            mine = g[self.rank]
            if self.r1 - self.r0 < self.per:
                mine[:, self.r1 - self.r0:].zero_()
            m = self.local.forward_out(x, delta, [mine.data_ptr()], ldy=self.per, col0=0, return_masks=return_masks)
            if self.world > 1:
                dist.all_gather_into_tensor(g.view(-1), mine.reshape(-1), group=self.group)
            full = y if y is not None else torch.empty((T, self.out), dtype=torch.bfloat16, device=x.device)
            if self.world * self.per == self.out:
                full.view(T, self.world, self.per).copy_(g.transpose(0, 1))
            else:
                full.copy_(g.transpose(0, 1).reshape(T, self.world * self.per)[:, :self.out])
        return (full, m) if return_masks else full

    def forward_host(self, x_host: torch.Tensor, delta: float, y_host: Optional[torch.Tensor] = None,
                     masks_host: Optional[torch.Tensor] = None) -> torch.Tensor:
        dev = torch.device("cuda", self.local.device)
        y, m = self.forward(x_host.to(dev, non_blocking=True), delta, return_masks=True)
        if y_host is None:
            y_host = torch.empty(y.shape, dtype=y.dtype)
        y_host.copy_(y)
        if masks_host is not None:
            masks_host.copy_(m)
        return y_host

    # bookkeeping delegated to this rank's layer (the all-gather is in our epilogue or NCCL's kernel)
    def score(self, x, stream=None):
        return self.local.score(x, stream)

    def last_launches(self) -> int:
        return self.local.last_launches()

    def last_plan(self) -> dict:
        return self.local.last_plan()

    def profile(self, enable: bool = True):
        self.local.profile(enable)

    def profile_read(self):
        return self.local.profile_read()


def token_range(T: int, rank: int, world: int):
    """Token-sharded prefill: this rank's [t0, t1)."""
    ranges, _ = balanced_ranges(T, world)
    return ranges[rank]
