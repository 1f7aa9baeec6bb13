"""Thin Python binding of libqtt.so (include/qtt.h) -- argument marshalling only.

Every step of the zip-up runs inside the CUDA library; this module only turns torch
tensors into the plain pointers / sizes of the C-ABI and back.  PyTorch is used for
device memory and streams.  There is no CPU fallback: if ``libqtt.so`` is missing or no
CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QTT_LIB", os.path.join(_HERE, "lib", "libqtt.so"))  # QTT_LIB: A/B variants in experiments

QTT_OK = 0
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ESHAPE", 3: "ECONFORM", 4: "ENUMERIC", 5: "ECAPACITY",
                6: "EGUARD", 7: "ECUDA", 8: "EUNSUPPORTED"}
NO_OPERATOR_ORTH = 1
WINDOW2 = 2                  # QTT_WINDOW2: super-core of two sites


class QttError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"qtt status {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Diag(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_void_p), ("sigma_stride", ctypes.c_int32), ("sweeps", ctypes.c_void_p),
                ("events", ctypes.POINTER(ctypes.c_void_p)), ("phase_cycles", ctypes.c_void_p)]


class _Trains(ctypes.Structure):
    _fields_ = [("n_sites", ctypes.c_int32), ("n_legs", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("d_out", ctypes.POINTER(ctypes.c_int32)), ("d_in", ctypes.POINTER(ctypes.c_int32)),
                ("ranks", ctypes.POINTER(ctypes.c_int32)), ("cores", ctypes.POINTER(ctypes.c_void_p)),
                ("dtype", ctypes.c_int32)]

QTT_F64, QTT_F32, QTT_C128 = 0, 1, 2


_lib = None

SYMBOLS = ["qtt_zipup_capacity", "qtt_zipup_workspace_bytes", "qtt_zipup_workspace_bytes_flags", "qtt_zipup",
           "qtt_zipup_summary", "qtt_variational_workspace_bytes", "qtt_variational",
           "qtt_variational_workspace_bytes_ex", "qtt_variational_ex",
           "qtt_zipup_sharded_sizes", "qtt_zipup_sharded",
           "qtt_round_capacity", "qtt_round_workspace_bytes", "qtt_round",
           "qtt_einsum_exact", "qtt_inner_workspace_bytes", "qtt_inner", "qtt_to_dense_workspace_bytes",
           "qtt_to_dense", "qtt_last_error", "qtt_version"]


def load_library(path: str = LIB_PATH):
    """Load libqtt.so and declare the C signatures (no GPU work)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    P = ctypes.POINTER(_Trains)
    vp, i32, f64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, ctypes.c_size_t
    L.qtt_zipup_capacity.argtypes = [ctypes.c_char_p, P, P, i32, ctypes.POINTER(i32)]
    L.qtt_zipup_capacity.restype = i32
    L.qtt_zipup_workspace_bytes.argtypes = [ctypes.c_char_p, P, P, P]
    L.qtt_zipup_workspace_bytes.restype = sz
    L.qtt_zipup_workspace_bytes_flags.argtypes = [ctypes.c_char_p, P, P, P, ctypes.c_uint32]
    L.qtt_zipup_workspace_bytes_flags.restype = sz
    L.qtt_zipup.argtypes = [ctypes.c_char_p, P, P, f64, i32, ctypes.c_uint32, P, vp, vp, vp, vp,
                            ctypes.POINTER(_Diag), vp, sz, vp]
    L.qtt_zipup.restype = i32
    L.qtt_variational_workspace_bytes.argtypes = [ctypes.c_char_p, P, P, P]
    L.qtt_variational_workspace_bytes.restype = sz
    L.qtt_variational.argtypes = [ctypes.c_char_p, P, P, P, vp, i32, vp, vp, vp, sz, vp]
    L.qtt_variational.restype = i32
    L.qtt_variational_workspace_bytes_ex.argtypes = [ctypes.c_char_p, P, P, P, i32]
    L.qtt_variational_workspace_bytes_ex.restype = sz
    L.qtt_variational_ex.argtypes = [ctypes.c_char_p, P, P, P, vp, P, vp, i32, i32, f64, i32, vp, vp, vp, sz, vp]
    L.qtt_variational_ex.restype = i32
    L.qtt_zipup_sharded_sizes.argtypes = [ctypes.c_char_p, P, P, i32, i32, i32, vp, vp, vp]
    L.qtt_zipup_sharded_sizes.restype = i32
    L.qtt_zipup_sharded.argtypes = [ctypes.c_char_p, P, P, f64, i32, ctypes.c_uint32, P, vp, vp, vp, vp, vp, i32,
                                    vp, vp, sz, vp]
    L.qtt_zipup_sharded.restype = i32
    L.qtt_zipup_summary.argtypes = [i32, i32, vp, vp, vp, vp, vp]
    L.qtt_zipup_summary.restype = i32
    L.qtt_round_capacity.argtypes = [P, i32, ctypes.POINTER(i32)]
    L.qtt_round_capacity.restype = i32
    L.qtt_round_workspace_bytes.argtypes = [P, i32]
    L.qtt_round_workspace_bytes.restype = sz
    L.qtt_round.argtypes = [P, vp, f64, i32, P, vp, vp, vp, vp, vp, sz, vp]
    L.qtt_round.restype = i32
    L.qtt_einsum_exact.argtypes = [ctypes.c_char_p, P, P, P, vp]
    L.qtt_einsum_exact.restype = i32
    L.qtt_inner_workspace_bytes.argtypes = [P, P]
    L.qtt_inner_workspace_bytes.restype = sz
    L.qtt_inner.argtypes = [P, P, vp, vp, sz, vp]
    L.qtt_inner.restype = i32
    L.qtt_to_dense_workspace_bytes.argtypes = [P]
    L.qtt_to_dense_workspace_bytes.restype = sz
    L.qtt_to_dense.argtypes = [P, ctypes.POINTER(i32), vp, ctypes.c_int64, vp, sz, vp]
    L.qtt_to_dense.restype = i32
    L.qtt_last_error.argtypes = []
    L.qtt_last_error.restype = ctypes.c_char_p
    L.qtt_version.argtypes = []
    L.qtt_version.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(st: int):
    if st != QTT_OK:
        raise QttError(st, _lib.qtt_last_error().decode())


def _stream_ptr(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


# ------------------------------------------------------------------------- trains

@dataclass
class DeviceTrains:
    """`batch` tensor trains of identical shape on the GPU.  cores[q] is a contiguous
    float64 CUDA tensor (B, r, d, r') or (B, w, d_out, d_in, w'); for outputs the bond
    sizes are capacities and member cores are packed at their actual ranks."""
    cores: List[torch.Tensor]
    ranks: List[int]
    d_out: List[int]
    d_in: Optional[List[int]] = None

    @property
    def n_sites(self) -> int:
        return len(self.cores)

    @property
    def n_legs(self) -> int:
        return 2 if self.d_in is not None else 1

    @property
    def batch(self) -> int:
        return int(self.cores[0].shape[0])

    @property
    def dtype_code(self) -> int:
        dt = self.cores[0].dtype
        return QTT_F32 if dt == torch.float32 else QTT_C128 if dt == torch.complex128 else QTT_F64

    def c_struct(self):
        L = self.n_sites
        keep = []
        d_out = (ctypes.c_int32 * L)(*self.d_out)
        d_in = (ctypes.c_int32 * L)(*self.d_in) if self.d_in is not None else None
        ranks = (ctypes.c_int32 * (L + 1))(*self.ranks)
        ptrs = (ctypes.c_void_p * L)(*[c.data_ptr() for c in self.cores])
        keep += [d_out, d_in, ranks, ptrs]
        s = _Trains(L, self.n_legs, self.batch, d_out,
                    ctypes.cast(d_in, ctypes.POINTER(ctypes.c_int32)) if d_in is not None else None,
                    ranks, ptrs, self.dtype_code)
        return s, keep


def to_device(cores_per_site: Sequence[np.ndarray], device="cuda", mpo: bool = False,
              dtype=np.float64) -> DeviceTrains:
    """Upload batch-stacked numpy cores: cores_per_site[q] has shape (B, r, d, r') (MPS)
    or (B, w, d_out, d_in, w') (MPO).  Single trains may be given without the batch axis.
    dtype np.float32 gives QTT_F32 trains (the fp32 variant of qtt_zipup), np.complex128
    QTT_C128 trains (the complex variant: the Fourier chain)."""
    cs = []
    for c in cores_per_site:
        c = np.asarray(c, dtype=dtype)
        want = 5 if mpo else 4
        if c.ndim == want - 1:
            c = c[None]
        cs.append(torch.from_numpy(np.ascontiguousarray(c)).to(device))
    ranks = [int(cs[0].shape[1])] + [int(c.shape[-1]) for c in cs]
    d_out = [int(c.shape[2]) for c in cs]
    d_in = [int(c.shape[3]) for c in cs] if mpo else None
    return DeviceTrains(cs, ranks, d_out, d_in)


def empty_like_capacity(batch: int, d_out: Sequence[int], cap: Sequence[int], device="cuda",
                        dtype=torch.float64) -> DeviceTrains:
    cores = [torch.zeros((batch, cap[q], d_out[q], cap[q + 1]), dtype=dtype, device=device)
             for q in range(len(d_out))]
    return DeviceTrains(cores, list(cap), list(d_out), None)


def member_cores(t: DeviceTrains, ranks: Sequence[int], b: int) -> List[np.ndarray]:
    """Unpack member b's cores (packed at `ranks` inside capacity slots) to numpy."""
    out = []
    for q, c in enumerate(t.cores):
        n = ranks[q] * t.d_out[q] * ranks[q + 1]
        flat = c[b].reshape(-1)[:n]
        flat = flat.cpu()
        flat = flat if flat.is_complex() else flat.double()
        out.append(flat.numpy().reshape(ranks[q], t.d_out[q], ranks[q + 1]))
    return out


def member_view(t: DeviceTrains, ranks: Sequence[int], b: int) -> DeviceTrains:
    """Member b of a capacity-sized output as a batch-1 train at its actual `ranks` (host
    ints): zero-copy views of the packed prefix of each slot, ready to feed the next call."""
    cores = []
    for q, c in enumerate(t.cores):
        n = ranks[q] * t.d_out[q] * ranks[q + 1]
        cores.append(c[b].reshape(-1)[:n].view(1, ranks[q], t.d_out[q], ranks[q + 1]))
    return DeviceTrains(cores, [int(r) for r in ranks], list(t.d_out), None)


# ------------------------------------------------------------------------- calls

@dataclass
class ZipupResult:
    out: DeviceTrains           # capacity-sized output cores
    ranks: torch.Tensor         # int32 (B, L+1) on device
    delta2: torch.Tensor        # float64 (B, L)
    norm2: torch.Tensor         # float64 (B,)
    status: torch.Tensor        # int32 (1,)
    sigma: Optional[torch.Tensor]  # float64 (B, L-1, sigma_stride) or None
    sweeps: Optional[torch.Tensor]  # int32 (B, L) Jacobi sweeps per site or None
    workspace: torch.Tensor
    cycles: Optional[torch.Tensor] = None  # int64 (B, L, 4) clock64 per site-kernel phase


def capacity(subscripts: str, op: Optional[DeviceTrains], x: DeviceTrains, max_rank: int) -> List[int]:
    L = load_library()
    xs, kx = x.c_struct()
    ops = None
    if op is not None:
        ops, ko = op.c_struct()
    cap = (ctypes.c_int32 * (x.n_sites + 1))()
    _check(L.qtt_zipup_capacity(subscripts.encode(), ctypes.byref(ops) if ops is not None else None,
                                ctypes.byref(xs), max_rank, cap))
    return list(cap)


class ZipupPlan:
    """Pre-allocated outputs + workspace for repeated qtt_zipup calls on fixed shapes
    (the bench loop and CUDA-graph capture use this; no allocation per call)."""

    def __init__(self, subscripts: str, op: Optional[DeviceTrains], x: DeviceTrains, eps: float,
                 max_rank: int, flags: int = 0, sigma_stride: int = 0, sweeps: bool = False, cycles: bool = False,
                 device="cuda"):
        self.lib = load_library()
        self.subscripts, self.eps, self.max_rank, self.flags = subscripts, float(eps), int(max_rank), int(flags)
        d_out = op.d_out if (op is not None and subscripts == "ij,j->i") else x.d_out
        self.cap = capacity(subscripts, op, x, max_rank)
        B, L = x.batch, x.n_sites
        self.out = empty_like_capacity(B, d_out, self.cap, device, dtype=x.cores[0].dtype)
        self.ranks = torch.zeros((B, L + 1), dtype=torch.int32, device=device)
        self.delta2 = torch.zeros((B, L), dtype=torch.float64, device=device)
        self.norm2 = torch.zeros((B,), dtype=torch.float64, device=device)
        self.status = torch.zeros((1,), dtype=torch.int32, device=device)
        self.sigma_stride = int(sigma_stride)
        self.sigma = (torch.zeros((B, max(L - 1, 1), sigma_stride), dtype=torch.float64, device=device)
                      if sigma_stride > 0 else None)
        self.sweeps = torch.zeros((B, L), dtype=torch.int32, device=device) if sweeps else None
        self.cycles = torch.zeros((B, L, 4), dtype=torch.int64, device=device) if cycles else None
        xs, kx = x.c_struct()
        os_ = None
        if op is not None:
            os_, ko = op.c_struct()
        outs, kout = self.out.c_struct()
        nbytes = self.lib.qtt_zipup_workspace_bytes_flags(subscripts.encode(),
                                                          ctypes.byref(os_) if os_ is not None else None,
                                                          ctypes.byref(xs), ctypes.byref(outs), self.flags)
        if nbytes == 0:
            raise QttError(2, self.lib.qtt_last_error().decode())
        self.workspace = torch.empty((nbytes + 255) // 256 * 256, dtype=torch.uint8, device=device)

    def run(self, op: Optional[DeviceTrains], x: DeviceTrains, stream=None, events=None) -> ZipupResult:
        """events: optional list of 4 torch.cuda.Event (a1 pre-pass start/end, sweep start/end)."""
        xs, kx = x.c_struct()
        os_ = None
        if op is not None:
            os_, ko = op.c_struct()
        outs, kout = self.out.c_struct()
        diag = None
        if self.sigma is not None or self.sweeps is not None or events is not None or self.cycles is not None:
            ev = None
            if events is not None:
                ev = (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])
            diag = _Diag(self.sigma.data_ptr() if self.sigma is not None else None, max(self.sigma_stride, 1),
                         self.sweeps.data_ptr() if self.sweeps is not None else None,
                         ctypes.cast(ev, ctypes.POINTER(ctypes.c_void_p)) if ev is not None else None,
                         self.cycles.data_ptr() if self.cycles is not None else None)
            self._keep = ev
        _check(self.lib.qtt_zipup(self.subscripts.encode(), ctypes.byref(os_) if os_ is not None else None,
                                  ctypes.byref(xs), self.eps, self.max_rank, self.flags, ctypes.byref(outs),
                                  self.ranks.data_ptr(), self.delta2.data_ptr(), self.norm2.data_ptr(),
                                  self.status.data_ptr(), ctypes.byref(diag) if diag is not None else None,
                                  self.workspace.data_ptr(), self.workspace.numel(), _stream_ptr(stream)))
        return ZipupResult(self.out, self.ranks, self.delta2, self.norm2, self.status, self.sigma, self.sweeps,
                           self.workspace, self.cycles)


class HostPipeline:
    """qtt_zipup on batches that live in (pinned) host memory, `depth` batches in flight.

    Buffer set i = k % depth holds batch k's device inputs and its ZipupPlan (outputs +
    workspace).  The host->device copy of batch k runs on a copy stream, the zip-up on the
    compute stream, the device->host copy of its results on a second copy stream; events
    order each set's reuse, so the copies of batches k+1 and k-1 overlap the zip-up of batch k.
    Host buffers given to step() must stay untouched until finish() (or the batch's d2h event).
    """

    def __init__(self, subscripts: str, op: Optional[DeviceTrains], x: DeviceTrains, eps: float,
                 max_rank: int, depth: int = 2, flags: int = 0, device="cuda"):
        def clone(t):
            return None if t is None else DeviceTrains([torch.empty_like(c) for c in t.cores], list(t.ranks),
                                                        list(t.d_out), None if t.d_in is None else list(t.d_in))
        self.sets = []
        for _ in range(depth):
            xi, oi = clone(x), clone(op)
            self.sets.append((oi, xi, ZipupPlan(subscripts, oi, xi, eps, max_rank, flags, device=device)))
        self.h2d = torch.cuda.Stream(device=device)
        self.d2h = torch.cuda.Stream(device=device)
        self.comp_done = [torch.cuda.Event() for _ in range(depth)]
        self.d2h_done = [torch.cuda.Event() for _ in range(depth)]
        self.used = [False] * depth
        self.k = 0

    def begin(self, stream=None):
        """Order both copy streams after everything already enqueued on `stream`."""
        s = stream if stream is not None else torch.cuda.current_stream()
        self.h2d.wait_stream(s)
        self.d2h.wait_stream(s)

    def step(self, host_x: Sequence[torch.Tensor], host_op: Optional[Sequence[torch.Tensor]],
             host_out: Sequence[torch.Tensor], host_ranks: torch.Tensor, host_delta2: torch.Tensor,
             host_norm2: torch.Tensor, stream=None) -> ZipupResult:
        s = stream if stream is not None else torch.cuda.current_stream()
        i = self.k % len(self.sets)
        op, x, plan = self.sets[i]
        with torch.cuda.stream(self.h2d):
            if self.used[i]:
                self.h2d.wait_event(self.comp_done[i])          # batch k-depth has read set i's inputs
            for dst, src in zip(x.cores, host_x):
                dst.copy_(src, non_blocking=True)
            if op is not None:
                for dst, src in zip(op.cores, host_op):
                    dst.copy_(src, non_blocking=True)
        s.wait_stream(self.h2d)
        if self.used[i]:
            s.wait_event(self.d2h_done[i])                      # batch k-depth's results are out
        res = plan.run(op, x, stream=s)
        self.comp_done[i].record(s)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.comp_done[i])
            for dst, src in zip(host_out, plan.out.cores):
                dst.copy_(src, non_blocking=True)
            host_ranks.copy_(res.ranks, non_blocking=True)
            host_delta2.copy_(res.delta2, non_blocking=True)
            host_norm2.copy_(res.norm2, non_blocking=True)
            self.d2h_done[i].record(self.d2h)
        self.used[i] = True
        self.k += 1
        return res

    def finish(self, stream=None):
        """Make `stream` wait for every outstanding device->host copy."""
        s = stream if stream is not None else torch.cuda.current_stream()
        s.wait_stream(self.d2h)


def zipup(subscripts: str, op: Optional[DeviceTrains], x: DeviceTrains, eps: float, max_rank: int,
          flags: int = 0, sigma_stride: int = 0, stream=None) -> ZipupResult:
    return ZipupPlan(subscripts, op, x, eps, max_rank, flags, sigma_stride, sweeps=True).run(op, x, stream)


def round_train(x: DeviceTrains, x_ranks: Optional[torch.Tensor], eps: float, max_rank: int,
                stream=None) -> ZipupResult:
    """qtt_round: right-to-left truncated-SVD sweep.  x_ranks: device int32
    (B, L+1) actual ranks of x's members (as qtt_zipup writes them), or None."""
    L = load_library()
    xs, kx = x.c_struct()
    cap = (ctypes.c_int32 * (x.n_sites + 1))()
    _check(L.qtt_round_capacity(ctypes.byref(xs), int(max_rank), cap))
    dev = x.cores[0].device
    out = empty_like_capacity(x.batch, x.d_out, list(cap), dev)
    os_, ko = out.c_struct()
    B, n = x.batch, x.n_sites
    ranks = torch.zeros((B, n + 1), dtype=torch.int32, device=dev)
    delta2 = torch.zeros((B, n), dtype=torch.float64, device=dev)
    norm2 = torch.zeros((B,), dtype=torch.float64, device=dev)
    status = torch.zeros((1,), dtype=torch.int32, device=dev)
    nbytes = L.qtt_round_workspace_bytes(ctypes.byref(xs), int(max_rank))
    ws = torch.empty(max(nbytes, 8), dtype=torch.uint8, device=dev)
    _check(L.qtt_round(ctypes.byref(xs), x_ranks.data_ptr() if x_ranks is not None else None, float(eps),
                       int(max_rank), ctypes.byref(os_), ranks.data_ptr(), delta2.data_ptr(), norm2.data_ptr(),
                       status.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
    return ZipupResult(out, ranks, delta2, norm2, status, None, None, ws)


@dataclass
class VariationalResult:
    out: DeviceTrains           # capacity-sized cores of C (centre at site 0)
    ranks: torch.Tensor         # int32 (B, L+1)
    center_norm2: torch.Tensor  # float64 (B, sweeps * 2L): |C_q|^2 after every update
    status: torch.Tensor


def variational(subscripts: str, op: Optional[DeviceTrains], x: DeviceTrains, seed: ZipupResult, sweeps: int,
                stream=None, ncores: int = 1, eps: float = 0.0, max_rank: int = 0,
                capacity: Optional[Sequence[int]] = None) -> VariationalResult:
    """qtt_variational_ex (f3): refine a zip-up result variationally.  The
    seed (the zip-up result) is read, not modified.  ncores = 2: two-site super-cores whose
    split is truncated by (eps, max_rank) -- ranks adapt up to the output capacity, by default
    min(max_rank, the digit products) per bond (gen-style clipping), else the seed's."""
    L = load_library()
    n = x.n_sites
    d = list(seed.out.d_out)
    if capacity is None:
        if ncores == 2:
            # the largest rank a split can keep at bond q: min(max_rank, the digit products on
            # either side, the bond of the exact product w_q r_q) -- and at least the seed's
            left, right = [1], [1]
            for q in range(n):
                left.append(left[-1] * d[q])
                right.append(right[-1] * d[n - 1 - q])
            exact = [a * b for a, b in zip(op.ranks, x.ranks)] if op is not None else list(x.ranks)
            capacity = []
            for q in range(n + 1):
                c = min(left[q], right[n - q], exact[q])
                if max_rank > 0:
                    c = min(c, max_rank)
                capacity.append(max(c, seed.out.ranks[q]))
        else:
            capacity = list(seed.out.ranks)
    dev = x.cores[0].device
    c = empty_like_capacity(x.batch, d, capacity, dev)
    ranks = torch.zeros_like(seed.ranks)
    xs, kx = x.c_struct()
    os_ = None
    if op is not None:
        os_, ko = op.c_struct()
    ss, ks = seed.out.c_struct()
    cs, kc = c.c_struct()
    B = x.batch
    norms = torch.zeros((B, sweeps * 2 * n), dtype=torch.float64, device=dev)
    status = torch.zeros((1,), dtype=torch.int32, device=dev)
    nbytes = L.qtt_variational_workspace_bytes_ex(subscripts.encode(),
                                                  ctypes.byref(os_) if os_ is not None else None,
                                                  ctypes.byref(xs), ctypes.byref(cs), int(ncores))
    if nbytes == 0:
        raise QttError(2, L.qtt_last_error().decode())
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _check(L.qtt_variational_ex(subscripts.encode(), ctypes.byref(os_) if os_ is not None else None,
                                ctypes.byref(xs), ctypes.byref(ss), seed.ranks.data_ptr(), ctypes.byref(cs),
                                ranks.data_ptr(), int(sweeps), int(ncores), float(eps), int(max_rank),
                                norms.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
    return VariationalResult(c, ranks, norms, status)


def summary(res: ZipupResult, stream=None) -> torch.Tensor:
    L = load_library()
    B, Lp1 = res.ranks.shape
    out = torch.zeros(4, dtype=torch.float64, device=res.ranks.device)
    _check(L.qtt_zipup_summary(B, Lp1 - 1, res.ranks.data_ptr(), res.delta2.data_ptr(), res.norm2.data_ptr(),
                               out.data_ptr(), _stream_ptr(stream)))
    return out


def einsum_exact(subscripts: str, a: DeviceTrains, b: DeviceTrains, stream=None) -> DeviceTrains:
    L = load_library()
    ranks = [x * y for x, y in zip(a.ranks, b.ranks)]
    out = empty_like_capacity(a.batch, a.d_out, ranks, a.cores[0].device)
    as_, ka = a.c_struct()
    bs, kb = b.c_struct()
    os_, ko = out.c_struct()
    _check(L.qtt_einsum_exact(subscripts.encode(), ctypes.byref(as_), ctypes.byref(bs), ctypes.byref(os_),
                              _stream_ptr(stream)))
    return out


def inner(a: DeviceTrains, b: DeviceTrains, stream=None) -> torch.Tensor:
    L = load_library()
    as_, ka = a.c_struct()
    bs, kb = b.c_struct()
    nbytes = L.qtt_inner_workspace_bytes(ctypes.byref(as_), ctypes.byref(bs))
    ws = torch.empty(max(nbytes, 8), dtype=torch.uint8, device=a.cores[0].device)
    res = torch.zeros(a.batch, dtype=torch.float64, device=a.cores[0].device)
    _check(L.qtt_inner(ctypes.byref(as_), ctypes.byref(bs), res.data_ptr(), ws.data_ptr(), ws.numel(),
                       _stream_ptr(stream)))
    return res


def to_dense(t: DeviceTrains, leg_dim: Optional[Sequence[int]] = None, max_elems: int = 0,
             stream=None) -> torch.Tensor:
    L = load_library()
    ts, kt = t.c_struct()
    N = int(np.prod(t.d_out))
    nbytes = L.qtt_to_dense_workspace_bytes(ctypes.byref(ts))
    ws = torch.empty(max(nbytes, 8), dtype=torch.uint8, device=t.cores[0].device)
    out = torch.empty((t.batch, N), dtype=torch.float64, device=t.cores[0].device)
    ld = (ctypes.c_int32 * t.n_sites)(*leg_dim) if leg_dim is not None else None
    _check(L.qtt_to_dense(ctypes.byref(ts), ld, out.data_ptr(), int(max_elems), ws.data_ptr(), ws.numel(),
                          _stream_ptr(stream)))
    return out
