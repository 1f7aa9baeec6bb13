"""The oracle result cache used by the full-size parity tests: round trip, and a cache written for
other inputs is never returned (its digest differs)."""
import numpy as np

import oracle_cache
from oracle.zipup import zipup
from paper_2602_20226_b200 import gen


def test_cache_round_trip_and_digest(tmp_path, monkeypatch):
    monkeypatch.setattr(oracle_cache, "CACHE", str(tmp_path / "cache"))
    monkeypatch.setattr(oracle_cache, "HERE", str(tmp_path))
    (tmp_path / "golden").mkdir()
    a = gen.random_mps([2] * 8, 6, np.random.default_rng(1)).cores
    b = gen.random_mps([2] * 8, 5, np.random.default_rng(2)).cores
    r1 = oracle_cache.oracle_result("t", "hadamard", a, b, 1e-6, 8)
    r2 = oracle_cache.oracle_result("t", "hadamard", a, b, 1e-6, 8)       # from the cache
    direct = zipup("hadamard", a, b, 1e-6, 8)
    assert r2["ranks"] == direct["ranks"] == r1["ranks"]
    for c2, cd in zip(r2["cores"], direct["cores"]):
        np.testing.assert_array_equal(c2, cd)
    np.testing.assert_array_equal(r2["sigmas"][3], direct["sigmas"][3])
    # other inputs under the same name: the stale cache is ignored
    b2 = [c.copy() for c in b]
    b2[0] = b2[0] * 2.0
    r3 = oracle_cache.oracle_result("t", "hadamard", a, b2, 1e-6, 8)
    assert abs(r3["norm"] - 2.0 * direct["norm"]) <= 1e-12 * r3["norm"]
    assert (tmp_path / "golden" / "t.json").exists()
