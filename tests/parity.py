"""GPU-vs-oracle comparison protocol (SURVEY.md §8(c) "Comparison protocol", c-A9, c-A28).

Gauge-invariant comparisons only (SVD signs are arbitrary, c-A8):
  1. bond ranks equal, except at *fragile* sites (near-ties at the cut), where the oracle
     is re-run with the GPU ranks forced;
  2. per-site singular values |s_G - s_O| <= stol * s_1 for j <= min(p, k+4);
  3. discarded mass delta2_q and ||y|| agree relative to ||T_q||^2 and ||y||;
  4. rel_fro(Y_G, Y_O) <= 1e-10 + eps (fp64), dense when small, else QR-sweep distance;
  5. four seeded rank-8 probe trains Z: |<Z,Y_G> - <Z,Y_O>| <= tol ||Z|| ||Y_O||.
"""
from __future__ import annotations

import math

import numpy as np

from oracle import tt
from oracle.zipup import zipup as oracle_zipup_w1, zipup_window

U64 = 1.1e-16


def fragile(sig: np.ndarray, k: int, eps: float, max_rank: int, u: float = U64) -> bool:
    """c-A9: the cut is within roundoff (unit roundoff u of the GPU dtype) of a decision boundary."""
    sig = np.asarray(sig)
    p = sig.size
    if p == 0:
        return False
    s1 = sig[0]
    slack = 10 * p * u * s1
    nrm = math.sqrt(float(np.sum(sig * sig)))
    for j in (k - 1, k):
        if 0 <= j <= p:
            tail = math.sqrt(float(np.sum(sig[j:] ** 2)))
            if abs(tail - eps * nrm) <= slack:
                return True
    if max_rank > 0 and k == max_rank and k < p and sig[k - 1] - sig[k] <= slack:
        return True
    return False


def probe_trains(x_cores, n=4, rank=8, seed=2602):
    """Protocol item 5: seeded rank-8 probe trains Z on the digit sizes of the result."""
    from paper_2602_20226_b200 import gen
    dims = [int(c.shape[1]) for c in x_cores]
    return [gen.random_mps(dims, rank, np.random.default_rng([seed, i])).cores for i in range(n)]


def compare(kind, op_cores, x_cores, eps, max_rank, gpu_cores, gpu_ranks, gpu_sigma, gpu_delta2, gpu_norm2,
            rel_tol=1e-10, sig_tol=1e-12, dense=True, orth_operator=True, u=U64, window=1, ref=None,
            probes=True):
    """Returns a dict of measured errors; raises AssertionError on a protocol violation.
    window: the zip-up super-core size the GPU ran with (1, or 2 for QTT_WINDOW2).
    ref: the oracle's result for these inputs when already computed (tests/oracle_cache.py)."""
    def oracle_zipup(*args, **kw):
        if window == 1:
            return oracle_zipup_w1(*args, **kw)
        return zipup_window(*args, window=window, **kw)

    if ref is None:
        ref = oracle_zipup(kind, op_cores, x_cores, eps, max_rank, orth_operator=orth_operator)
    L = len(x_cores)
    if list(gpu_ranks) != ref["ranks"]:
        for q in range(L - 1):
            if gpu_ranks[q + 1] != ref["ranks"][q + 1]:
                assert fragile(ref["sigmas"][q], ref["ranks"][q + 1], eps, max_rank, u), \
                    f"rank mismatch at bond {q + 1}: gpu {list(gpu_ranks)} oracle {ref['ranks']}"
        ref = oracle_zipup(kind, op_cores, x_cores, eps, max_rank, force_ranks=list(gpu_ranks),
                           orth_operator=orth_operator)
    out = {"ranks": list(gpu_ranks)}
    # 2. singular values
    worst = 0.0
    if gpu_sigma is not None:
        for q in range(L - 1):
            so = ref["sigmas"][q]
            k = ref["ranks"][q + 1]
            n = min(so.size, k + 4, gpu_sigma.shape[-1])
            if so.size == 0 or so[0] == 0:
                continue
            err = float(np.max(np.abs(gpu_sigma[q][:n] - so[:n]))) / so[0]
            worst = max(worst, err)
        assert worst <= sig_tol, f"singular values differ by {worst:.3e} * s_1"
    out["sigma_err"] = worst
    # 3. discarded mass and norm
    werr = 0.0
    for q in range(L - 1):
        t2 = float(np.sum(ref["sigmas"][q] ** 2))
        if t2 > 0:
            werr = max(werr, abs(gpu_delta2[q] - ref["delta2"][q]) / t2)
    d2_tol = 1e-12 if rel_tol <= 1e-9 else rel_tol          # fp64 / fp32 variant (c-A28)
    assert werr <= d2_tol, f"delta2 differs by {werr:.3e} of ||T||^2"
    out["delta2_err"] = werr
    ny = ref["norm"]
    nerr = abs(math.sqrt(max(gpu_norm2, 0.0)) - ny) / max(ny, 1e-300)
    assert nerr <= 1e-12 + rel_tol, f"norm differs by {nerr:.3e}"
    out["norm_err"] = nerr
    # 4. the result itself
    if dense:
        yg, yo = tt.to_dense_vector(gpu_cores), tt.to_dense_vector(ref["cores"])
        rel = float(np.linalg.norm(yg - yo) / max(np.linalg.norm(yo), 1e-300))
    else:
        rel = tt.diff_norm(gpu_cores, ref["cores"]) / max(tt.qr_norm(ref["cores"]), 1e-300)
    assert rel <= rel_tol + eps, f"rel_fro {rel:.3e} > {rel_tol + eps:.1e}"
    out["rel_fro"] = rel
    # 5. seeded probe inner products |<Z, Y_G> - <Z, Y_O>| <= tol ||Z|| ||Y_O||
    if probes:
        worst_p = 0.0
        for Z in probe_trains(ref["cores"]):
            zn = tt.qr_norm(Z)
            dv = abs(tt.inner(Z, gpu_cores) - tt.inner(Z, ref["cores"])) / max(zn * ny, 1e-300)
            worst_p = max(worst_p, dv)
        assert worst_p <= rel_tol + eps, f"probe inner products differ by {worst_p:.3e}"
        out["probe_err"] = worst_p
    out["ref"] = ref
    return out
