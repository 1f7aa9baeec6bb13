"""CPU oracle for the zip-up hot path of arXiv 2602.20226 (trainsum).

TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct float64 NumPy code that
follows the paper step by step.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  The
product path (``paper_2602_20226_b200`` + ``libqtt.so``) never imports, links or
calls anything here, and this package imports nothing from the product path
except the seeded input generators (``paper_2602_20226_b200.gen``, which hold no
zip-up arithmetic).

Modules
  tt.py     exact train algebra: dense conversion, inner products, exact addition
            (PAPER.md:196-209), exact einsum (Eq. einsum),
            QR normalisation, QR-sweep norms, TT-SVD, rounding.
  zipup.py  the decomposition / zip-up algorithm with window N=1,
            SVD by LAPACK directly on each site matrix, truncation rule SPEC.md:299.

Parity status: every function is pinned by ``tests/test_oracle_*.py`` against closed
forms, dense brute force or proven identities.
The only unpinned behaviour is the *bare* zip-up rank trajectory of general MPO
products, which is algorithm-defined (SURVEY.md c-A12): "parity unpinned" for the
exact rank numbers of that case; its values are pinned through the eps->0 limit,
the orthogonal-operator / sign-Hadamard TT-SVD identities and the error bounds.
"""
