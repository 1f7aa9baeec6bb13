"""CPU-side checks of the boundary: the library loads and exports every symbol that
include/qtt.h declares, and host-only entry points validate their arguments
(no GPU work is issued here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qtt.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qtt_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("qtt_zipup", "qtt_einsum_exact", "qtt_inner", "qtt_to_dense"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2602_20226_b200 import qtt
    if not os.path.exists(qtt.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    lib = qtt.load_library()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(qtt.SYMBOLS) == declared_symbols()
    assert b"sm_100a" in lib.qtt_version()


def _mps_struct(qtt, dims, ranks, batch=1):
    L = len(dims)
    d = (ctypes.c_int32 * L)(*dims)
    r = (ctypes.c_int32 * (L + 1))(*ranks)
    p = (ctypes.c_void_p * L)(*([1] * L))   # never dereferenced by host-only calls
    return qtt._Trains(L, 1, batch, d, None, r, p), (d, r, p)


def test_capacity_and_validation_host_only():
    from paper_2602_20226_b200 import qtt
    lib = qtt.load_library()
    x, kx = _mps_struct(qtt, [2] * 6, [1, 2, 4, 8, 4, 2, 1])
    cap = (ctypes.c_int32 * 7)()
    assert lib.qtt_zipup_capacity(b"i->i", None, ctypes.byref(x), 3, cap) == 0
    assert list(cap) == [1, 2, 3, 3, 3, 2, 1]
    assert lib.qtt_zipup_capacity(b"i->i", None, ctypes.byref(x), 0, cap) == 0
    assert list(cap) == [1, 2, 4, 8, 4, 2, 1]
    # Hadamard of two trains: cap[q+1] = min(cap[q]*d, a'*b') (bare zip-up ranks may exceed
    # the minimal ones, SURVEY.md c-A12)
    assert lib.qtt_zipup_capacity(b"i,i->i", ctypes.byref(x), ctypes.byref(x), 0, cap) == 0
    assert list(cap) == [1, 2, 4, 8, 16, 4, 1]
    # unsupported subscripts / bad boundary ranks / conformance
    assert lib.qtt_zipup_capacity(b"ij,jk->ik", ctypes.byref(x), ctypes.byref(x), 0, cap) == 8
    bad, kb = _mps_struct(qtt, [2] * 6, [2, 2, 4, 8, 4, 2, 1])
    assert lib.qtt_zipup_capacity(b"i->i", None, ctypes.byref(bad), 0, cap) == 2
    y, ky = _mps_struct(qtt, [3] * 6, [1, 2, 4, 8, 4, 2, 1])
    assert lib.qtt_zipup_capacity(b"i,i->i", ctypes.byref(y), ctypes.byref(x), 0, cap) == 3
    assert b"misaligned" in lib.qtt_last_error()
    assert lib.qtt_zipup_workspace_bytes(b"i->i", None, ctypes.byref(x), None) > 0


def test_to_dense_guard_host_only():
    from paper_2602_20226_b200 import qtt
    lib = qtt.load_library()
    x, kx = _mps_struct(qtt, [2] * 25, [1] + [2] * 24 + [1])
    out = ctypes.c_void_p(1)
    st = lib.qtt_to_dense(ctypes.byref(x), None, out, 0, None, 0, None)
    assert st == 6 and b"guard" in lib.qtt_last_error()   # 2^25 > 2^24 (SURVEY c-A30)


def test_sharded_and_variational_ex_validation_host_only():
    """qtt_zipup_sharded(_sizes) and qtt_variational_ex refuse bad arguments before any GPU
    work (SURVEY.md §8(f) f3/f4 entry points; qtt.h error conventions)."""
    from paper_2602_20226_b200 import qtt
    from paper_2602_20226_b200.shard import _Comm, _ALLGATHER
    lib = qtt.load_library()
    x, kx = _mps_struct(qtt, [2] * 6, [1, 2, 4, 8, 4, 2, 1])
    r_el, c_el, wsb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    assert lib.qtt_zipup_sharded_sizes(b"i,i->i", ctypes.byref(x), ctypes.byref(x), 0, 2, 2, ctypes.byref(r_el),
                                       ctypes.byref(c_el), ctypes.byref(wsb)) == 0
    assert r_el.value >= 1 and c_el.value >= 1 and wsb.value > 0
    xb, kxb = _mps_struct(qtt, [2] * 6, [1, 2, 4, 8, 4, 2, 1], batch=2)
    assert lib.qtt_zipup_sharded_sizes(b"i,i->i", ctypes.byref(xb), ctypes.byref(xb), 0, 2, 1, ctypes.byref(r_el),
                                       ctypes.byref(c_el), ctypes.byref(wsb)) == 8        # batch != 1
    assert lib.qtt_zipup_sharded_sizes(b"i,i->i", ctypes.byref(x), ctypes.byref(x), 0, 0, 1, ctypes.byref(r_el),
                                       ctypes.byref(c_el), ctypes.byref(wsb)) == 1        # world 0
    one = ctypes.c_void_p(1)
    comm = _Comm(2, 0, 1, _ALLGATHER(), None, 1, 1, 1, 1)                                # world 2, no callback
    st = lib.qtt_zipup_sharded(b"i,i->i", ctypes.byref(x), ctypes.byref(x), 1e-8, 0, ctypes.c_uint32(0),
                               ctypes.byref(x), one, one, one, one, None, 1, ctypes.byref(comm), one, 1 << 30, None)
    assert st == 1 and b"callback" in lib.qtt_last_error()
    comm = _Comm(1, 3, 1, _ALLGATHER(), None, 1, 1, 1, 1)                                # rank outside [0, world)
    st = lib.qtt_zipup_sharded(b"i,i->i", ctypes.byref(x), ctypes.byref(x), 1e-8, 0, ctypes.c_uint32(0),
                               ctypes.byref(x), one, one, one, one, None, 1, ctypes.byref(comm), one, 1 << 30, None)
    assert st == 1 and b"rank" in lib.qtt_last_error()
    st = lib.qtt_zipup_sharded(b"i,i->i", ctypes.byref(x), ctypes.byref(x), 1e-8, 0, ctypes.c_uint32(2),
                               ctypes.byref(x), one, one, one, one, None, 1, ctypes.byref(comm), one, 1 << 30, None)
    assert st == 8                                                                        # QTT_WINDOW2
    # qtt_variational_ex: ncores must be 1 or 2; the output capacity must hold the seed
    st = lib.qtt_variational_ex(b"i->i", None, ctypes.byref(x), ctypes.byref(x), one, ctypes.byref(x), one, 1, 3,
                                0.0, 0, one, one, one, 1 << 30, None)
    assert st == 8 and b"ncores" in lib.qtt_last_error()
    small, ks = _mps_struct(qtt, [2] * 6, [1, 2, 2, 2, 2, 2, 1])
    st = lib.qtt_variational_ex(b"i->i", None, ctypes.byref(x), ctypes.byref(x), one, ctypes.byref(small), one, 1, 2,
                                0.0, 0, one, one, one, 1 << 30, None)
    assert st == 5 and b"capacity" in lib.qtt_last_error()
    assert lib.qtt_variational_workspace_bytes_ex(b"i->i", None, ctypes.byref(x), ctypes.byref(x), 2) > 0
    assert lib.qtt_variational_workspace_bytes_ex(b"i->i", None, ctypes.byref(x), ctypes.byref(x), 4) == 0
