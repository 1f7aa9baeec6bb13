"""On-disk cache of oracle zip-up results for the full-size parity tests (test infrastructure).

A cached result is written only by `oracle.zipup` (this module or the committed script
scripts/make_oracle_golden.py, which calls this module) -- never from the CUDA path.  The key
is a SHA-256 digest of the operand cores and the zip-up parameters, so a stale cache (other
inputs, other generator) is ignored and recomputed.  The .npz files live under
tests/golden/cache/ (git-ignored: tens of MB of fp64 cores); the small committed summary
tests/golden/<name>.json (ranks, delta^2, norm, leading singular values, digest) documents
the run and lets a test check that a cache matches what the committed script produced.
"""
from __future__ import annotations

import hashlib
import json
import os
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.path.join(HERE, "golden", "cache")


def digest(kind, op, x, eps, max_rank, window=1):
    h = hashlib.sha256()
    h.update(f"{kind}|{eps!r}|{max_rank}|{window}".encode())
    for group in (op or []), x:
        for c in group:
            a = np.ascontiguousarray(c)
            h.update(str(a.dtype).encode() + str(a.shape).encode())
            h.update(a.tobytes())
    return h.hexdigest()


def _load(path, dg):
    try:
        z = np.load(path, allow_pickle=False)
    except (OSError, ValueError):
        return None
    if str(z["digest"]) != dg:
        return None
    L = int(z["L"])
    ranks = [int(v) for v in z["ranks"]]
    return {"cores": [z[f"core{q}"] for q in range(L)], "ranks": ranks,
            "delta2": [float(v) for v in z["delta2"]],
            "sigmas": [z[f"sig{q}"] for q in range(L - 1)], "norm": float(z["norm"]), "digest": dg}


def summary(ref, dg, seconds):
    return {"digest": dg, "ranks": ref["ranks"], "delta2": ref["delta2"], "norm": ref["norm"],
            "sigma_head": [[float(v) for v in s[:4]] for s in ref["sigmas"]],
            "sigma_at_cut": [[float(v) for v in s[max(0, k - 2):k + 4]] for s, k in zip(ref["sigmas"], ref["ranks"][1:])],
            "oracle_seconds": round(seconds, 1)}


def oracle_result(name, kind, op, x, eps, max_rank, window=1, write=True):
    """The oracle's zip-up of (op, x): from tests/golden/cache/<name>.npz when its digest matches,
    else computed by oracle.zipup (and cached when write)."""
    from oracle.zipup import zipup, zipup_window
    dg = digest(kind, op, x, eps, max_rank, window)
    path = os.path.join(CACHE, name + ".npz")
    ref = _load(path, dg)
    if ref is not None:
        return ref
    t0 = time.perf_counter()
    if window == 1:
        ref = zipup(kind, op, x, eps, max_rank)
    else:
        ref = zipup_window(kind, op, x, eps, max_rank, window=window)
    dt = time.perf_counter() - t0
    ref["digest"] = dg
    if write:
        os.makedirs(CACHE, exist_ok=True)
        L = len(ref["cores"])
        arrs = {f"core{q}": c for q, c in enumerate(ref["cores"])}
        arrs.update({f"sig{q}": s for q, s in enumerate(ref["sigmas"])})
        tmp = path + ".tmp.npz"
        np.savez(tmp, digest=np.array(dg), L=np.array(L), ranks=np.array(ref["ranks"]),
                 delta2=np.array(ref["delta2"]), norm=np.array(ref["norm"]), **arrs)
        os.replace(tmp, path)
        with open(os.path.join(HERE, "golden", name + ".json"), "w") as f:
            json.dump(summary(ref, dg, dt), f, indent=1)
    return ref
