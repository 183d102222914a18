"""NEXT-4: one filter problem sharded across GPUs in slabs, with a halo exchange.

Partition (host, deterministic on every rank from the same centroids): slabs along the longest
bounding-box axis, cut at the coordinate quantiles (balanced by point count; equal coordinates
stay together). Rank k owns the points of its slab and needs, as halo, every other rank's point
within rmin of the slab (coordinate in [lo_k - rmin, hi_k + rmin)): an owned point's neighbours
all lie in owned + halo, so the owned rows of a filter built on (owned + halo) centroids are the
global rows (same pairs, same fp64 weights; columns in local order, so sums differ from the
unsharded filter only by summation order). Slabs thinner than rmin simply draw halo from more
ranks.

Per apply: pack the owned values each other rank needs (tf_halo_pack, a library kernel),
exchange them point-to-point (torch.distributed batch_isend_irecv: NCCL over NVLink/NVSwitch
on GPUs; x and dc land directly in the halo tail of the local vectors, no unpack), run the
library filter's owned rows (tf_*_filter_rows: the local order puts them first) on the local
vectors, and return them. The exchange is the path's one
real collective step; everything else is the single-GPU library.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np


@dataclass
class ShardPlan:
    """Partition metadata of one rank (host arrays of global ids, all sorted ascending)."""
    rank: int
    world: int
    axis: int
    bounds: np.ndarray                       # [world+1] slab bounds along `axis` (-inf, ..., +inf)
    owned: np.ndarray                        # global ids owned by this rank
    halo_from: dict = field(default_factory=dict)  # src rank -> global ids received (in order)
    send_to: dict = field(default_factory=dict)    # dst rank -> LOCAL indices (into owned) sent

    @property
    def n_owned(self) -> int:
        return int(self.owned.shape[0])

    @property
    def n_halo(self) -> int:
        return int(sum(v.shape[0] for v in self.halo_from.values()))

    def local_ids(self) -> np.ndarray:
        """Global ids of the local vector: owned, then each source rank's halo in rank order."""
        parts = [self.owned] + [self.halo_from[j] for j in sorted(self.halo_from)]
        return np.concatenate(parts) if parts else np.zeros(0, np.int64)

    def halo_offset(self, src: int) -> int:
        off = self.n_owned
        for j in sorted(self.halo_from):
            if j == src:
                return off
            off += self.halo_from[j].shape[0]
        raise KeyError(src)


def slab_partition(c: np.ndarray, world: int, rmin: float, axis: int | None = None):
    """Owner rank of every point and the slab bounds (see module docstring)."""
    c = np.asarray(c, dtype=np.float64)
    n = c.shape[0]
    if axis is None:
        axis = int(np.argmax(c.max(axis=0) - c.min(axis=0))) if n else 0
    coord = c[:, axis]
    srt = np.sort(coord, kind="stable")
    cuts = [srt[(k * n) // world] for k in range(1, world)] if n else [0.0] * (world - 1)
    bounds = np.array([-np.inf] + list(cuts) + [np.inf])
    owner = np.searchsorted(np.asarray(cuts), coord, side="right").astype(np.int64)
    return owner, bounds, axis


def make_plans(c: np.ndarray, world: int, rmin: float, axis: int | None = None) -> list[ShardPlan]:
    """ShardPlan of every rank (each rank may compute all and keep its own)."""
    c = np.asarray(c, dtype=np.float64)
    owner, bounds, axis = slab_partition(c, world, rmin, axis)
    coord = c[:, axis]
    ids = np.arange(c.shape[0], dtype=np.int64)
    owned = [ids[owner == k] for k in range(world)]
    plans = [ShardPlan(k, world, axis, bounds, owned[k]) for k in range(world)]
    for k in range(world):
        lo, hi = bounds[k] - rmin, bounds[k + 1] + rmin
        need = (coord >= lo) & (coord < hi) & (owner != k)
        for j in np.unique(owner[need]):
            j = int(j)
            g = ids[need & (owner == j)]
            plans[k].halo_from[j] = g
            # rank j sends these, in this order, as local indices into its owned array
            plans[j].send_to[k] = np.searchsorted(owned[j], g).astype(np.int32)
    return plans


class DistTransport:
    """Point-to-point exchange over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, sends: dict, recvs: dict):
        """sends: dst -> list of tensors; recvs: src -> list of tensors (filled in place)."""
        dist = self.dist
        ops = []
        for dst, ts in sorted(sends.items()):
            ops += [dist.P2POp(dist.isend, t, dst, self.group) for t in ts]
        for src, ts in sorted(recvs.items()):
            ops += [dist.P2POp(dist.irecv, t, src, self.group) for t in ts]
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()


class ShardedFilter:
    """This rank's shard of a filter over the global centroids (NEXT-4)."""

    def __init__(self, centroids, rmin: float, rank: int, world: int, transport=None, axis: int | None = None,
                 plan: ShardPlan | None = None, device=None):
        import torch
        import paper_2012_08208_b200 as tf
        self.tf = tf
        c = np.asarray(centroids, dtype=np.float64)
        self.plan = plan if plan is not None else make_plans(c, world, rmin, axis)[rank]
        self.rank, self.world = rank, world
        self.transport = transport
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        loc = self.plan.local_ids()
        self.n_local = int(loc.shape[0])
        self.filter = tf.tf_build_filter(torch.from_numpy(np.ascontiguousarray(c[loc])).to(self.device), rmin)
        self.send_idx = {j: torch.from_numpy(v).to(self.device) for j, v in self.plan.send_to.items()}
        self.x_loc = torch.empty(self.n_local, dtype=torch.float64, device=self.device)
        self.dc_loc = torch.empty(self.n_local, dtype=torch.float64, device=self.device)
        self.out_loc = torch.empty(self.n_local, dtype=torch.float64, device=self.device)
        self.out2_loc = torch.empty(self.n_local, dtype=torch.float64, device=self.device)

    # -- pieces (also used by in-process emulation) -------------------------------------------
    def pack(self, x_owned, dc_owned=None) -> dict:
        """dst -> [x values(, dc values)] this rank sends (packed by the library kernel)."""
        import torch
        out = {}
        stream = torch.cuda.current_stream(self.device)
        for j, idx in self.send_idx.items():
            bufs = []
            for src in ([x_owned] if dc_owned is None else [x_owned, dc_owned]):
                b = torch.empty(idx.shape[0], dtype=torch.float64, device=self.device)
                self.tf._check(self.tf.lib().tf_halo_pack(ctypes.c_void_p(src.data_ptr()),
                                                          ctypes.c_void_p(idx.data_ptr()), idx.shape[0],
                                                          ctypes.c_void_p(b.data_ptr()),
                                                          ctypes.c_void_p(stream.cuda_stream)))
                bufs.append(b)
            out[j] = bufs
        return out

    def recv_views(self, with_dc: bool) -> dict:
        """src -> views of the local vectors' halo segments (receive targets)."""
        v = {}
        for j, g in self.plan.halo_from.items():
            o = self.plan.halo_offset(j)
            m = g.shape[0]
            v[j] = [self.x_loc[o:o + m]] + ([self.dc_loc[o:o + m]] if with_dc else [])
        return v

    def _fill_owned(self, x_owned, dc_owned):
        n = self.plan.n_owned
        self.x_loc[:n].copy_(x_owned)
        if dc_owned is not None:
            self.dc_loc[:n].copy_(dc_owned)

    # -- applies -------------------------------------------------------------------------------
    def _exchange(self, x_owned, dc_owned):
        import torch
        self._fill_owned(x_owned, dc_owned)
        sends = self.pack(x_owned, dc_owned)
        torch.cuda.current_stream(self.device).synchronize()  # packed buffers complete before NCCL reads them
        self.transport.exchange(sends, self.recv_views(dc_owned is not None))

    def sensitivity(self, x_owned, dc_owned):
        """Owned rows of the sensitivity filter (Eq. filter)."""
        self._exchange(x_owned, dc_owned)
        self.filter.sensitivity(self.x_loc, self.dc_loc, out=self.out_loc, rows=self.plan.n_owned)
        return self.out_loc[:self.plan.n_owned]

    def density(self, x_owned):
        self._exchange(x_owned, None)
        self.filter.density(self.x_loc, out=self.out_loc, rows=self.plan.n_owned)
        return self.out_loc[:self.plan.n_owned]

    def apply_with_halo(self, x_owned, dc_owned, received: dict, density: bool = False):
        """In-process emulation: the halo values `received` (src -> [x, dc]) are copied in."""
        self._fill_owned(x_owned, dc_owned)
        for j, bufs in received.items():
            for dstv, b in zip(self.recv_views(dc_owned is not None)[j], bufs):
                dstv.copy_(b)
        n = self.plan.n_owned  # the owned rows come first in the local order; halo rows are not needed
        if density:
            self.filter.density(self.x_loc, out=self.out_loc, rows=n)
        else:
            self.filter.sensitivity(self.x_loc, self.dc_loc, out=self.out_loc, rows=n)
        return self.out_loc[:self.plan.n_owned]

    def close(self):
        self.filter.close()
