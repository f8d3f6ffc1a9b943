"""Victim selection (sine_select_victims, csrc/select.cuh) against the
oracle's order on the device store: every policy, ascending and shuffled
ids, tombstoned rows, unpurged expired rows (LCFU score 0), heavy key ties
(integer created_at, LFU's small frequencies) and excesses from one token
to more than the whole store.  The expected list is the reference's
`_victim_order_locked` (engine.py:369-383: ascending (key, created_at, id))
cut where the size sum first reaches the excess (the pop loops at
engine.py:321-327, :353-359).  A lowered shared-memory cap drives the
single-CTA, bucketed and merge (oversized bucket) paths on small stores."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import sine_oracle as O

pytestmark = pytest.mark.gpu

POLICY = {"lcfu": 0, "lru": 1, "lfu": 2}


@pytest.fixture(scope="module")
def pkg():
    import paper_2509_17360_b200 as P
    from paper_2509_17360_b200 import _native as N
    if N.device_count() < 1:
        pytest.skip("no CUDA device")
    return P


def _meta(n, seed, tied):
    rng = np.random.default_rng(seed)
    m = dict(staticity=rng.integers(1, 11, n), freq=rng.integers(0, 8, n),
             lat=rng.choice(np.array([50.0, 400.0, 1500.0]), n),
             cost=rng.choice(np.array([0.0, 0.0005, 0.005, 0.02]), n), size=rng.integers(1, 30, n))
    m["created"] = rng.integers(0, 40, n).astype(np.float64) if tied else rng.random(n) * 1e4
    m["last_access"] = m["created"] + (rng.integers(0, 5, n) if tied else rng.random(n) * 10)
    ttl = np.where(rng.random(n) < 1 / 7, 5.0, 2.0e4)
    m["expiration"] = m["created"] + ttl
    return m


def _store(pkg, ids, m):
    import torch

    n = ids.shape[0]
    cols = {"log_freq": O._exact_log((m["freq"] + 1).astype(np.float64)),
            "log_cost": O._exact_log(m["cost"] * 1000.0 + 1), "log_lat": O._exact_log(m["lat"] + 1),
            "log_stat": O._exact_log((m["staticity"] + 1).astype(np.float64)),
            "frequency": m["freq"], "size_tokens": m["size"], "created_at": m["created"],
            "expiration_time": m["expiration"], "last_access": m["last_access"]}
    rows = torch.zeros((n, 4), dtype=torch.float64, device="cuda")
    rows[:, 0] = 1.0
    idx = pkg.GpuCosineIndex(4, metadata=True, capacity=n)
    idx.insert_device(ids, rows.data_ptr(), meta=cols)
    return idx


def _order(policy, ids, m, now, live):
    if policy == "lcfu":
        key = O.lcfu_scores_np(m["freq"], m["cost"], m["lat"], m["staticity"], m["size"], m["expiration"], now)
    elif policy == "lru":
        key = m["last_access"].astype(np.float64)
    else:
        key = m["freq"].astype(np.float64)
    sel = np.nonzero(live)[0]
    o = np.lexsort((ids[sel], m["created"][sel], key[sel]))
    return sel[o]


def _select(idx, policy, now, excess, n):
    from paper_2509_17360_b200 import _native as N

    out = np.empty(max(n, 1), dtype=np.int64)
    cnt = ctypes.c_int64()
    N.check(idx._lib.sine_select_victims(idx.handle, POLICY[policy], now, int(excess), N.ptr(out, ctypes.c_int64),
                                         out.shape[0], ctypes.byref(cnt)))
    return out[:cnt.value].copy()


@pytest.mark.parametrize("shuffled", [False, True])
@pytest.mark.parametrize("tied", [False, True])
def test_select_matches_oracle_order(pkg, shuffled, tied):
    from paper_2509_17360_b200 import _native as N

    n = 300_000
    m = _meta(n, 5 + shuffled + 2 * tied, tied)
    rng = np.random.default_rng(3)
    ids = (rng.permutation(3 * n)[:n] + 1) if shuffled else np.arange(1, n + 1)
    idx = _store(pkg, ids, m)
    # tombstones: 2% of the rows removed (below the compaction threshold)
    dead = rng.choice(n, n // 50, replace=False)
    idx.remove_batch(ids[dead])
    live = np.ones(n, dtype=bool)
    live[dead] = False
    now = 20.0
    total = int(m["size"][live].sum())
    for cap in (6144, 512):
        N.check(idx._lib.sine_set_select_cap(idx.handle, cap))
        for policy in ("lcfu", "lru", "lfu"):
            order = _order(policy, ids, m, now, live)
            cum = np.cumsum(m["size"][order])
            for excess in (1, 29, total // 10_000, total // 10, total // 2, total - 1, total, total + 7):
                if excess <= 0:
                    continue
                want = ids[order[:int(np.searchsorted(cum, excess, side="left")) + 1]]
                got = _select(idx, policy, now, excess, n)
                assert np.array_equal(got, want), (cap, policy, excess, got.shape, want.shape)


def test_select_small_store_and_edges(pkg):
    """Stores below the sample threshold (every slot a record), a single
    live row, excess beyond everything, and an empty store."""
    n = 3000
    m = _meta(n, 11, True)
    ids = np.arange(10, 10 + n)
    idx = _store(pkg, ids, m)
    live = np.ones(n, dtype=bool)
    for policy in ("lcfu", "lru", "lfu"):
        order = _order(policy, ids, m, 3.0, live)
        cum = np.cumsum(m["size"][order])
        for excess in (1, 1000, int(cum[-1]), int(cum[-1]) + 1):
            want = ids[order[:int(np.searchsorted(cum, excess, side="left")) + 1]]
            assert np.array_equal(_select(idx, policy, 3.0, excess, n), want)
    idx.remove_batch(ids[1:])
    assert _select(idx, "lcfu", 3.0, 10**9, n).tolist() == [int(ids[0])]
    idx.remove_batch(ids[:1])
    assert _select(idx, "lcfu", 3.0, 5, n).tolist() == []


def test_select_merge_path_large(pkg):
    """2M rows with the cap at 64: every bucket above the cap goes through
    the chunk-sort + merge-path kernel, including the cut bucket."""
    from paper_2509_17360_b200 import _native as N

    n = 2_000_000
    m = _meta(n, 21, False)
    ids = np.arange(1, n + 1)
    idx = _store(pkg, ids, m)
    N.check(idx._lib.sine_set_select_cap(idx.handle, 64))
    live = np.ones(n, dtype=bool)
    order = _order("lcfu", ids, m, 50.0, live)
    cum = np.cumsum(m["size"][order])
    for excess in (int(cum[-1]) // 3, int(cum[-1]) // 3 * 2):
        want = ids[order[:int(np.searchsorted(cum, excess, side="left")) + 1]]
        assert np.array_equal(_select(idx, "lcfu", 50.0, excess, n), want)
