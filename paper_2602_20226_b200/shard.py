"""Cross-GPU sharding of ONE zip-up (qtt.h qtt_zipup_sharded).

The library drives the site loop; between the steps of every site it calls back into Python
to all-gather two things over torch.distributed (NCCL over NVLink on the B200 box, gloo in
the CPU tests): phase 0 -- each shard's m x m column-slab factor F_t (the R-tree input: the R
of the stacked factors is the R of T^H), phase 1 -- each shard's carry slab U_k^T T_t (the
carry exchange).  This module holds only that plumbing: the shard ranges, the exchange
buffers and the all-gather callback.  All arithmetic runs in libqtt.so.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Tuple

import torch


def shard_range(n: int, S: int, t: int) -> Tuple[int, int]:
    """Contiguous balanced range of shard t of S over n columns (the library's shard_range)."""
    return (t * n) // S, ((t + 1) * n) // S


class ShardExchange:
    """Send / receive buffers of the two per-site exchanges and the all-gather itself.
    recv[rank * local_shards + s] = send[s] of every rank (shard order = rank-major)."""

    def __init__(self, world: int, rank: int, local_shards: int, r_elems: int, c_elems: int, device,
                 dist=None, group=None):
        self.world, self.rank, self.ls = int(world), int(rank), int(local_shards)
        self.r_elems, self.c_elems = int(r_elems), int(c_elems)
        self.dist, self.group = dist, group
        dt = torch.float64
        self.send_r = torch.zeros(self.ls * self.r_elems, dtype=dt, device=device)
        self.recv_r = torch.zeros(self.world * self.ls * self.r_elems, dtype=dt, device=device)
        self.send_c = torch.zeros(self.ls * self.c_elems, dtype=dt, device=device)
        self.recv_c = torch.zeros(self.world * self.ls * self.c_elems, dtype=dt, device=device)
        self.calls: List[int] = []

    def allgather(self, phase: int) -> None:
        send, recv = (self.send_r, self.recv_r) if phase == 0 else (self.send_c, self.recv_c)
        self.calls.append(int(phase))
        if self.world == 1 or self.dist is None:
            recv[self.rank * send.numel():(self.rank + 1) * send.numel()].copy_(send)
            return
        self.dist.all_gather_into_tensor(recv, send, group=self.group)


_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p)


class _Comm(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("local_shards", ctypes.c_int32),
                ("allgather", _ALLGATHER), ("user", ctypes.c_void_p),
                ("send_r", ctypes.c_void_p), ("recv_r", ctypes.c_void_p),
                ("send_c", ctypes.c_void_p), ("recv_c", ctypes.c_void_p)]


def zipup_sharded(subscripts: str, op, x, eps: float, max_rank: int, world: int = 1, rank: int = 0,
                  local_shards: int = 1, dist=None, group=None, sigma_stride: int = 0, flags: int = 0,
                  stream=None, callback: Optional[bool] = None):
    """qtt_zipup_sharded: this process's part of one zip-up split into world * local_shards
    column shards.  Returns (ZipupResult, ShardExchange).  Every process gets the full
    output (identical values)."""
    from . import qtt
    L = qtt.load_library()
    xs, kx = x.c_struct()
    os_ = None
    if op is not None:
        os_, ko = op.c_struct()
    r_el, c_el, wsb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    qtt._check(L.qtt_zipup_sharded_sizes(subscripts.encode(), ctypes.byref(os_) if os_ is not None else None,
                                         ctypes.byref(xs), int(max_rank), int(world), int(local_shards),
                                         ctypes.byref(r_el), ctypes.byref(c_el), ctypes.byref(wsb)))
    dev = x.cores[0].device
    ex = ShardExchange(world, rank, local_shards, r_el.value, c_el.value, dev, dist, group)
    d_out = op.d_out if (op is not None and subscripts == "ij,j->i") else x.d_out
    cap = qtt.capacity(subscripts, op, x, max_rank)
    n = x.n_sites
    out = qtt.empty_like_capacity(1, d_out, cap, dev)
    ranks = torch.zeros((1, n + 1), dtype=torch.int32, device=dev)
    delta2 = torch.zeros((1, n), dtype=torch.float64, device=dev)
    norm2 = torch.zeros((1,), dtype=torch.float64, device=dev)
    status = torch.zeros((1,), dtype=torch.int32, device=dev)
    sigma = (torch.zeros((1, max(n - 1, 1), sigma_stride), dtype=torch.float64, device=dev)
             if sigma_stride > 0 else None)
    ws = torch.empty(max(int(wsb.value), 256), dtype=torch.uint8, device=dev)
    errors: List[BaseException] = []

    def cb(phase, user):
        try:
            ex.allgather(int(phase))
            return 0
        except BaseException as e:           # never let an exception cross the C frame
            errors.append(e)
            return 1

    use_cb = (world > 1 or dist is not None) if callback is None else bool(callback)
    cfun = _ALLGATHER(cb) if use_cb else _ALLGATHER()
    comm = _Comm(int(world), int(rank), int(local_shards), cfun, None, ex.send_r.data_ptr(),
                 ex.recv_r.data_ptr(), ex.send_c.data_ptr(), ex.recv_c.data_ptr())
    outs, kout = out.c_struct()
    st = L.qtt_zipup_sharded(subscripts.encode(), ctypes.byref(os_) if os_ is not None else None, ctypes.byref(xs),
                             float(eps), int(max_rank), ctypes.c_uint32(flags), ctypes.byref(outs), ranks.data_ptr(),
                             delta2.data_ptr(), norm2.data_ptr(), status.data_ptr(),
                             sigma.data_ptr() if sigma is not None else None, int(max(sigma_stride, 1)),
                             ctypes.byref(comm), ws.data_ptr(), ws.numel(), qtt._stream_ptr(stream))
    if errors:
        raise errors[0]
    qtt._check(st)
    return qtt.ZipupResult(out, ranks, delta2, norm2, status, sigma, None, ws), ex
