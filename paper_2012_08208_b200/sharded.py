"""NEXT-4: one filter problem sharded over GPUs in slabs with a
point-to-point halo exchange.

Plan: `tf_shard_plan` (library, on the device; include/topofilt.h) cuts slabs along the longest
bounding-box axis at count quantiles and returns this rank's local order
[interior | boundary | halo by source rank] (global ids) and its send lists (local indices). The
rank gathers its local centroids with `tf_gather_rows` and builds an ordinary library filter on
them: the owned rows are the global rows (same pairs, bitwise the same fp64 weights; columns in
local order, so sums differ from the unsharded filter only by summation order).

Per apply (everything on the caller's current CUDA stream, no host synchronisation):
  1. x (and dc) of the owned points go into the local vectors; the values other ranks need are
     packed by `tf_halo_pack` (library kernel) into one contiguous send buffer per destination;
  2. the exchange is posted (`transport.exchange`: `torch.distributed.batch_isend_irecv`, NCCL
     over NVLink/NVSwitch; NCCL's stream waits for the packs, the call returns at once);
  3. the INTERIOR rows (no halo column) are filtered while the exchange is in flight
     (`tf_*_filter_range`, rows [0, n_interior));
  4. `wait()` orders the compute stream after the exchange; the received values are copied into
     the halo tail of the local vectors and the BOUNDARY rows are filtered
     (rows [n_interior, n_owned)).
The exchange is the path's one real collective step; everything else is the single-GPU library.
`LoopbackTransport` runs W shards as threads of one process on one GPU (tests, dry runs).
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np


class ShardPlan:
    """This rank's slab (owns a tf_shard handle): sizes, local ids, send lists, counts."""

    def __init__(self, centroids, rmin: float, world: int, rank: int, stream=None):
        import torch
        import paper_2012_08208_b200 as tf
        self.tf = tf
        c = centroids
        if not (isinstance(c, torch.Tensor) and c.is_cuda and c.dtype == torch.float64 and c.dim() == 2):
            raise TypeError("centroids must be a CUDA float64 [n, dim] tensor")
        c = c.contiguous()
        self.device = c.device
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            tf._check(tf.lib().tf_shard_plan(ctypes.c_void_p(c.data_ptr()), c.shape[0], c.shape[1], float(rmin),
                                             int(world), int(rank), tf._stream_ptr(stream, self.device),
                                             ctypes.byref(h)))
        self._h = h
        v = tf.tf_shard_view()
        tf._check(tf.lib().tf_shard_view_get(h, ctypes.byref(v)))
        self.world, self.rank, self.axis = v.nranks, v.rank, v.axis
        self.cut_lo, self.cut_hi = v.cut_lo, v.cut_hi
        self.n_interior, self.n_owned, self.n_halo = v.n_interior, v.n_owned, v.n_halo
        self.n_local = self.n_owned + self.n_halo
        recv = (ctypes.c_int64 * world)()
        send = (ctypes.c_int64 * world)()
        tf._check(tf.lib().tf_shard_counts(h, recv, send))
        self.recv = [int(r) for r in recv]
        self.send = [int(s) for s in send]
        mk = lambda p, n: torch.as_tensor(tf._CudaArray(p, (n,), "<i4"), device=self.device)  # noqa: E731
        self.local_ids = mk(v.local_ids, self.n_local) if self.n_local else torch.zeros(0, dtype=torch.int32,
                                                                                         device=self.device)
        ns = sum(self.send)
        self.send_idx = mk(v.send_idx, ns) if ns else torch.zeros(0, dtype=torch.int32, device=self.device)

    @property
    def owned_ids(self):
        """Global ids of the owned points in the shard's owned order ([interior | boundary])."""
        return self.local_ids[:self.n_owned]

    def halo_range(self, src: int):
        """[start, end) of the halo received from rank src inside the local order."""
        o = self.n_owned + sum(self.recv[:src])
        return o, o + self.recv[src]

    def send_range(self, dst: int):
        o = sum(self.send[:dst])
        return o, o + self.send[dst]

    def close(self):
        if self._h is not None:
            self.tf.lib().tf_shard_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistTransport:
    """Point-to-point exchange over torch.distributed (NCCL on GPUs, gloo on CPU tensors).
    exchange() posts the ops and returns at once; wait() orders the current stream after them."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, sends: dict, recvs: dict):
        """sends: dst -> tensor; recvs: src -> tensor (filled). Returns a handle with wait()."""
        dist = self.dist
        ops = [dist.P2POp(dist.isend, t, dst, self.group) for dst, t in sorted(sends.items())]
        ops += [dist.P2POp(dist.irecv, t, src, self.group) for src, t in sorted(recvs.items())]
        works = dist.batch_isend_irecv(ops) if ops else []

        class _H:
            def wait(self_inner):
                for w in works:
                    w.wait()  # NCCL: a stream dependency, not a host block
        return _H()


class LoopbackTransport:
    """W shards as threads of one process (one GPU): exchange() is a barrier-synchronised copy from
    the senders' buffers. The sender's stream is synchronised before its buffers are published, so
    no kernel ever waits on another thread's kernel (tests and dry runs only)."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.box = {}

    def endpoint(self, rank: int):
        return _LoopbackEndpoint(self, rank)


class _LoopbackEndpoint:
    def __init__(self, hub: LoopbackTransport, rank: int):
        self.hub, self.rank = hub, rank

    def exchange(self, sends: dict, recvs: dict):
        import torch
        torch.cuda.current_stream().synchronize()  # packed buffers complete before peers read them
        for dst, t in sends.items():
            self.hub.box[(self.rank, dst)] = t
        self.hub.barrier.wait()
        for src, t in recvs.items():
            t.copy_(self.hub.box[(src, self.rank)])
        torch.cuda.current_stream().synchronize()
        self.hub.barrier.wait()  # every peer has copied before buffers are reused
        if self.rank == 0:
            self.hub.box.clear()
        self.hub.barrier.wait()

        class _H:
            def wait(self_inner):
                pass
        return _H()


class ShardedFilter:
    """This rank's shard of a filter over the global centroids (NEXT-4). Inputs and outputs are
    the owned points' values in the shard's owned order (ShardPlan.owned_ids)."""

    def __init__(self, centroids, rmin: float, rank: int, world: int, transport=None, stream=None):
        import torch
        import paper_2012_08208_b200 as tf
        self.tf = tf
        self.rank, self.world = rank, world
        self.transport = transport
        self.plan = ShardPlan(centroids, rmin, world, rank, stream)
        self.device = self.plan.device
        p = self.plan
        dim = centroids.shape[1]
        with torch.cuda.device(self.device):
            local_c = torch.empty(p.n_local, dim, dtype=torch.float64, device=self.device)
            if p.n_local:
                tf.tf_gather_rows(centroids.contiguous(), p.local_ids, local_c, stream)
            self.filter = tf.tf_build_filter(local_c, rmin) if p.n_owned else None
            del local_c
            z = lambda n: torch.empty(n, dtype=torch.float64, device=self.device)  # noqa: E731
            self.x_loc, self.dc_loc, self.out_loc = z(p.n_local), z(p.n_local), z(p.n_local)
            ns, nr = sum(p.send), p.n_halo
            self.sbuf, self.rbuf = z(2 * ns), z(2 * nr)  # [x | dc] per destination / source

    # -- exchange ---------------------------------------------------------------------------------
    def _post(self, x_owned, dc_owned):
        """Owned values into the local vectors, pack the sends, post the exchange."""
        tf, p = self.tf, self.plan
        n = p.n_owned
        self.x_loc[:n].copy_(x_owned)
        if dc_owned is not None:
            self.dc_loc[:n].copy_(dc_owned)
        k = 2 if dc_owned is not None else 1
        sends, recvs = {}, {}
        stream = tf._stream_ptr(None, self.device)
        for j in range(self.world):
            s0, s1 = p.send_range(j)
            if s1 > s0:
                buf = self.sbuf[k * s0:k * s1]
                idx = p.send_idx[s0:s1]
                for u, src in enumerate((self.x_loc, self.dc_loc)[:k]):
                    tf._check(tf.lib().tf_halo_pack(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(idx.data_ptr()),
                                                    s1 - s0, ctypes.c_void_p(buf.data_ptr() + 8 * u * (s1 - s0)),
                                                    stream))
                sends[j] = buf
            h0, h1 = p.halo_range(j)
            if h1 > h0:
                o0, o1 = h0 - n, h1 - n
                recvs[j] = self.rbuf[k * o0:k * o1]
        return self.transport.exchange(sends, recvs), recvs, k

    def _land(self, recvs, k):
        """Received values into the halo tail of the local vectors (stream-ordered copies)."""
        p = self.plan
        for j, buf in recvs.items():
            h0, h1 = p.halo_range(j)
            m = h1 - h0
            self.x_loc[h0:h1].copy_(buf[:m])
            if k == 2:
                self.dc_loc[h0:h1].copy_(buf[m:2 * m])

    # -- applies ----------------------------------------------------------------------------------
    def sensitivity(self, x_owned, dc_owned):
        """Owned rows of the sensitivity filter (Eq. filter)."""
        import torch
        tf, p = self.tf, self.plan
        with torch.cuda.device(self.device):
            h, recvs, k = self._post(x_owned, dc_owned)
            if p.n_interior:  # overlaps the exchange
                tf.tf_sensitivity_filter_range(self.filter, self.x_loc, self.dc_loc, self.out_loc, 0, p.n_interior)
            h.wait()
            self._land(recvs, k)
            if p.n_owned > p.n_interior:
                tf.tf_sensitivity_filter_range(self.filter, self.x_loc, self.dc_loc, self.out_loc, p.n_interior,
                                               p.n_owned)
        return self.out_loc[:p.n_owned]

    def density(self, x_owned):
        import torch
        tf, p = self.tf, self.plan
        with torch.cuda.device(self.device):
            h, recvs, k = self._post(x_owned, None)
            if p.n_interior:
                tf.tf_density_filter_range(self.filter, self.x_loc, self.out_loc, 0, p.n_interior)
            h.wait()
            self._land(recvs, k)
            if p.n_owned > p.n_interior:
                tf.tf_density_filter_range(self.filter, self.x_loc, self.out_loc, p.n_interior, p.n_owned)
        return self.out_loc[:p.n_owned]

    def close(self):
        if self.filter is not None:
            self.filter.close()
            self.filter = None
        self.plan.close()
