"""Native host RNG runtime (libskg) vs numpy: stream derivation and batch selection."""

import ctypes as C

import numpy as np
import pytest

import skewgcn_oracle as O
from paper_2101_07706_b200 import pcg64_state
from paper_2101_07706_b200._native import check, lib, ptr
from paper_2101_07706_b200.seeding import generator_state


@pytest.mark.parametrize("seed,labels", [
    (0, ("plan", 0, 1, 2)), (0, ("batch", 3, 17, 7)), (12345678901234567, ("init", 4)),
    (2 ** 64 - 1, ("partition",)), (7, ()), (1 << 40, ("x", -3, "y")), (0, ("sbm-edges",)),
])
def test_spawn_pcg64_matches_numpy(seed, labels):
    st, _, _ = generator_state(O.spawn_rng(seed, *labels))
    np.testing.assert_array_equal(pcg64_state(seed, *labels), st)


def _choice_native(rng, pop, size):
    st, has, u = generator_state(rng)
    out = np.zeros(max(size, 1), dtype=np.int64)
    check(lib.skg_choice_noreplace(ptr(st, C.c_uint64), has, u, pop, size, ptr(out, C.c_int64)))
    return np.sort(out[:size])


@pytest.mark.parametrize("pop,size", [(5, 3), (100, 100), (9999, 512), (10001, 199), (10001, 201),
                                      (19213, 512), (20000, 400), (20000, 401), (1, 1), (50, 0),
                                      (300000, 6001), (300000, 4500)])
def test_choice_without_replacement(pop, size):
    for seed in range(5):
        a = np.sort(np.random.default_rng(seed).choice(pop, size=size, replace=False))
        b = _choice_native(np.random.default_rng(seed), pop, size)
        np.testing.assert_array_equal(a, b)


def test_choice_with_buffered_uint32():
    # a generator holding a buffered 32-bit half must use it first (pcg64_next32)
    rng = np.random.default_rng(3)
    rng.integers(0, 10, size=1, dtype=np.uint32)
    a = np.sort(np.random.default_rng(3).choice(1000, 10, replace=False))  # noqa: F841
    r2 = np.random.default_rng(3)
    r2.integers(0, 10, size=1, dtype=np.uint32)
    st = generator_state(r2)
    b = _choice_native(r2, 1000, 10)
    r3 = np.random.default_rng(3)
    r3.integers(0, 10, size=1, dtype=np.uint32)
    np.testing.assert_array_equal(np.sort(r3.choice(1000, 10, replace=False)), b)
    assert st[1] in (0, 1)


@pytest.mark.parametrize("n_train,bs", [(19213, 512), (474, 512), (8000, 512), (30, 8), (60000, 512)])
def test_iteration_inputs_match_reference_loop(n_train, bs):
    train_w = np.sort(np.random.default_rng(n_train).choice(10 ** 6, n_train, replace=False)).astype(np.int64)
    for (seed, epoch, it, w) in [(0, 0, 0, 0), (11, 2, 37, 5), (2 ** 40 + 3, 9, 1, 7)]:
        brng = O.spawn_rng(seed, "batch", epoch, it, w)
        take = min(bs, n_train)
        exp = O.node_set(brng.choice(train_w, size=take, replace=False))
        exp_state, _, _ = generator_state(O.spawn_rng(seed, "plan", epoch, it, w))
        out = np.zeros(take, dtype=np.int64)
        n = C.c_int64()
        st = np.zeros(4, dtype=np.uint64)
        check(lib.skg_iteration_inputs(seed, epoch, it, w, ptr(train_w, C.c_int64), n_train, bs,
                                       ptr(out, C.c_int64), C.byref(n), ptr(st, C.c_uint64)))
        np.testing.assert_array_equal(out[: n.value], exp)
        np.testing.assert_array_equal(st, exp_state)


def test_group_inputs_equal_per_iteration_calls():
    """skg_group_inputs (a look-ahead group's host work on a thread pool) == the
    per-iteration skg_iteration_inputs calls, item by item."""
    import ctypes as C
    from paper_2101_07706_b200._native import check, lib, ptr
    rng = np.random.default_rng(3)
    tws = [np.sort(rng.choice(50_000, int(rng.integers(300, 4000)), replace=False)).astype(np.int64)
           for _ in range(6)]
    n = 18
    ep = rng.integers(0, 3, n).astype(np.int64)
    its = rng.integers(0, 50, n).astype(np.int64)
    ws = rng.integers(0, 6, n).astype(np.int32)
    ptrs = np.array([tws[w].ctypes.data for w in ws], dtype=np.uint64)
    lens = np.array([len(tws[w]) for w in ws], dtype=np.int64)
    bs = 512
    bids = np.zeros(n * bs, dtype=np.int64)
    boff = np.zeros(n + 1, dtype=np.int64)
    st = np.zeros((n, 4), dtype=np.uint64)
    check(lib.skg_group_inputs(11, n, ptr(ep, C.c_int64), ptr(its, C.c_int64), ptr(ws, C.c_int32),
                               ptr(ptrs, C.c_uint64), ptr(lens, C.c_int64), bs, ptr(bids, C.c_int64),
                               ptr(boff, C.c_int64), ptr(st, C.c_uint64), 4))
    b1 = np.zeros(bs, dtype=np.int64)
    s1 = np.zeros(4, dtype=np.uint64)
    ln = C.c_int64()
    for i in range(n):
        check(lib.skg_iteration_inputs(11, int(ep[i]), int(its[i]), int(ws[i]), ptr(tws[ws[i]], C.c_int64),
                                       len(tws[ws[i]]), bs, ptr(b1, C.c_int64), C.byref(ln),
                                       ptr(s1, C.c_uint64)))
        np.testing.assert_array_equal(bids[boff[i]:boff[i + 1]], b1[:ln.value])
        np.testing.assert_array_equal(st[i], s1)
