"""Pins of the oracle's steepest single-flip descent (oracle.descend, reading R-search in DESIGN.md
§3): against an independent walk over the EXHAUSTIVE key table of small random traces (every
mask's key computed once by index; the neighbour of mask m across item k is m ^ 2^k), the
defining properties of its end point (no single flip improves it; keys fall strictly along the
path), and its special cases (max_rounds = 0, a start at the global optimum).  The device
descent (chm_descend) is compared with this oracle in tests/test_gpu_descend.py."""
import numpy as np
import pytest

import oracle as O
from workloads import traces as W


def _table(m):
    """(excess, stall, swapped) of all 2^K masks, by mask index (EXHAUSTIVE kind, §8(c).4)"""
    r = m.eval(O.EXHAUSTIVE, 0, 1 << m.K, nthreads=8)
    ex = np.maximum(r["peak"] - m.trace.budget, 0)
    return ex, r["stall"], r["swapped"]


def _walk(tab, K, start, max_rounds=4096):
    """steepest descent over the table: argmin of (excess, stall, swapped, k) over the K
    neighbours, move while its first three fields are smaller"""
    ex, st, sw = tab
    key = lambda i: (int(ex[i]), float(st[i]), int(sw[i]))  # noqa: E731
    cur, rounds = start, 0
    while rounds < max_rounds:
        k = min(range(K), key=lambda j: key(cur ^ (1 << j)) + (j,))
        if not key(cur ^ (1 << k)) < key(cur):
            break
        cur ^= 1 << k
        rounds += 1
    return cur, key(cur), rounds


def _mask_index(words, K):
    return sum(1 << k for k in range(K) if (int(words[k // 64]) >> (k % 64)) & 1)


def _trace(seed):
    return W.random_trace(seed, n_layers=5, ops_per_layer=4, bw=3e7, t_iter=1e-3)


SEEDS = [200, 201, 202, 203, 207, 212]  # K = 12 .. 16


@pytest.mark.parametrize("seed", SEEDS)
def test_descend_equals_the_walk_over_the_exhaustive_table(seed):
    m = O.Model(_trace(seed))
    assert 12 <= m.K <= 16
    tab = _table(m)
    rng = np.random.default_rng(seed)
    starts = [0, (1 << m.K) - 1, _mask_index(m.base_mask(), m.K)] + [int(x) for x in rng.integers(0, 1 << m.K, 3)]
    for s in starts:
        words = np.array([s], np.uint64)
        e, key, r = O.descend(m, words, nthreads=2)
        ws, wkey, wr = _walk(tab, m.K, s)
        assert (_mask_index(e, m.K), key, r) == (ws, wkey, wr), (s, key, wkey)


@pytest.mark.parametrize("seed", SEEDS[:3])
def test_descend_start_at_the_optimum_and_zero_rounds(seed):
    m = O.Model(_trace(seed))
    ex, st, sw = _table(m)
    opt = min(range(1 << m.K), key=lambda i: (int(ex[i]), float(st[i]), int(sw[i]), i))
    e, key, r = O.descend(m, np.array([opt], np.uint64), nthreads=2)
    assert r == 0 and _mask_index(e, m.K) == opt
    s = int(np.random.default_rng(seed).integers(0, 1 << m.K))
    e, key, r = O.descend(m, np.array([s], np.uint64), max_rounds=0, nthreads=2)
    assert r == 0 and _mask_index(e, m.K) == s and key == (int(ex[s]), float(st[s]), int(sw[s]))


def test_descend_end_is_a_single_flip_local_minimum_on_c5():
    """C5 (K = 472): the end point of the descent from the argmax-window base is a strict local
    minimum of (excess, stall, swapped) over single flips, and the path only went down"""
    m = O.Model(W.CONFIGS["C5"]())
    b = m.base_mask()
    k0 = m.eval(O.MASKS, 0, 1, words=b)["best"]
    e, key, r = O.descend(m, b)
    assert r > 0 and key < (int(k0.excess), float(k0.stall), int(k0.swapped))
    nb = np.repeat(e[None, :], m.K, axis=0)
    for k in range(m.K):
        nb[k, k // 64] ^= np.uint64(1 << (k % 64))
    res = m.eval(O.MASKS, 0, m.K, words=nb.reshape(-1), nthreads=16)
    ex = np.maximum(res["peak"] - m.trace.budget, 0)
    for k in range(m.K):
        assert not (int(ex[k]), float(res["stall"][k]), int(res["swapped"][k])) < key
