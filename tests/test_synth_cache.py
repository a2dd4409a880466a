"""The versioned workload cache (synth/cache.py) returns exactly the generator's arrays, reloads
them from disk, and keys on every config field (no method arithmetic involved)."""
import dataclasses

import numpy as np

import synth
from synth import cache


def test_cache_roundtrip(tmp_path, monkeypatch):
    monkeypatch.setenv("MAYURA_WORKLOAD_CACHE", str(tmp_path))
    cfg = synth.CONFIGS["C1"]
    ref = cfg.generate()
    a = cache.cached(cfg)                     # generates + writes
    assert len(list(tmp_path.glob("*.json"))) == 1
    b = cache.cached(cfg)                     # loads
    for x, y, z in zip(ref[:3], a[:3], b[:3]):
        assert x.dtype == y.dtype == z.dtype and np.array_equal(x, y) and np.array_equal(x, z)
    assert ref[3] == a[3] == b[3]
    other = dataclasses.replace(cfg, seed=cfg.seed + 1)
    assert cache.key(other) != cache.key(cfg)
    c = cache.cached(other)
    assert not np.array_equal(c[2], ref[2])
    assert len(list(tmp_path.glob("*.json"))) == 2


def test_cache_rejects_corrupt_header(tmp_path, monkeypatch):
    monkeypatch.setenv("MAYURA_WORKLOAD_CACHE", str(tmp_path))
    cfg = synth.CONFIGS["C1"]
    cache.cached(cfg)
    hdr = next(tmp_path.glob("*.json"))
    hdr.write_text(hdr.read_text().replace('"format": 1', '"format": 0'))
    again = cache.cached(cfg)                 # stale header: regenerated, not trusted
    assert np.array_equal(again[0], cfg.generate()[0])
