"""CPU: host-side logic of the product library (no GPU needed).

- libatmgrit.so loads and exports every symbol include/atmgrit.h declares
- rank layout / per-rank ranges restate runtime/layout.cpp and parallel.cpp
  (tests/test_runtime.cpp:17-192 of the reference)
- the direct window-payload schedule delivers exactly the union of each
  rank's local windows, the set the reference's two-round group exchange
  delivers (parallel.cpp:134-194)
- the product path fails loudly without a GPU (no CPU fallback)
"""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2107_09596_b200 as T
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "atmgrit.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(atm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    out = subprocess.check_output(["nm", "-D", "--defined-only", T.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert T.lib().atm_abi_version() == 6


def test_python_binding_covers_the_abi():
    from paper_2107_09596_b200._capi import SIGNATURES
    assert set(declared_symbols()) <= set(SIGNATURES)


def test_host_random_state_matches_oracle():
    for seed, n in ((0, 5), (20, 63), (12345, 4095)):
        assert np.array_equal(T.random_state(seed, n), O.random_state(seed, n))


def test_gpu_path_fails_loudly_without_device():
    if T.lib().atm_device_count() > 0:
        pytest.skip("a GPU is present")
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 33), [4], 3)
    with pytest.raises(T.RuntimeFault):
        T.CycleDriver(T.Dahlquist(), hier, T.SolverConfig())


def test_config_errors_before_any_device_work():
    with pytest.raises(T.ConfigError):
        T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 5), [1], 2)
    with pytest.raises(T.ConfigError):
        T.TimeGrid.make(0.0, 1.0, 1)
    with pytest.raises(T.ConfigError):
        T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 3), [4], 2)
    # heat1d rows: one CTA up to 5376 unknowns, a cluster of up to 16 past that
    hier = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 33), [4], 3)
    with pytest.raises(T.ConfigError, match="65536"):
        T.CycleDriver(T.Heat1D(65537, manufactured_forcing=False), hier, T.SolverConfig())


# ---------------------------------------------------------------- grids

def test_hierarchy_windows_fig1():
    # test_grids.cpp:10-30
    h = T.build_hierarchy(T.TimeGrid.make(0.0, 15.0, 16), [2], 4)
    assert h.n_coarsest_points() == 8
    assert h.level(1).dt == pytest.approx(2.0)
    assert (h.local_grid(5).lo, h.local_grid(5).size()) == (2, 4)
    assert (h.local_grid(7).lo, h.local_grid(7).size()) == (4, 4)
    sp = T.make_cf_split(16, 2)
    assert len(sp.c_points) == 8 and len(sp.intervals) == 8
    h3 = T.build_hierarchy(T.TimeGrid.make(0.0, 20.0, 21), [2, 2], 4)
    assert [h3.level(l).n_points for l in range(3)] == [21, 11, 6]


# ---------------------------------------------------------------- layout

def test_layout_one_point_per_rank():
    # test_runtime.cpp:17-38
    h = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 18), [3], 3)
    lay = T.build_layout(h, 6)
    assert lay.coarse_lo == list(range(6)) and lay.coarse_hi == list(range(6))
    assert (lay.fine_lo[0], lay.fine_hi[0]) == (0, 0)
    assert (lay.fine_lo[1], lay.fine_hi[1]) == (1, 3)
    assert (lay.fine_lo[4], lay.fine_hi[4]) == (10, 12)
    assert (lay.fine_lo[5], lay.fine_hi[5]) == (13, 17)


def test_layout_rejects_too_many_workers_and_tiles_contiguously():
    h = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 18), [3], 3)
    with pytest.raises(T.ConfigError):
        T.build_layout(h, 7)
    h2 = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, 40), [3], 2)
    for p in range(1, h2.n_coarsest_points() + 1):
        lay = T.build_layout(h2, p)
        nxt = 0
        for r in range(p):
            assert lay.fine_lo[r] == nxt
            nxt = lay.fine_hi[r] + 1
        assert nxt == 40


def test_balance_within_one_interval():
    # test_runtime.cpp:294-312
    h = T.build_hierarchy(T.TimeGrid.make(0.0, 64.0, 512), [16], 16)
    lay = T.build_layout(h, 8)
    calls = [0] * 8
    for (c, first, last) in h.split(0).intervals:
        owner = next(r for r in range(8) if lay.fine_lo[r] <= first <= lay.fine_hi[r])
        calls[owner] += last - first + 1
    mean = sum(calls) / 8
    assert all(abs(c - mean) <= 15 + 1e-9 for c in calls)


def _ranges_reference(h, lay, rank):
    """parallel.cpp:67-130 restated independently in Python."""
    L = h.n_levels()
    out = {k: [] for k in ("lo", "hi", "iv_first", "iv_count", "c_first", "c_count")}
    stride = 1
    for l in range(L):
        n_l = h.level(l).n_points
        lo = -(-lay.fine_lo[rank] // stride)
        hi = min(lay.fine_hi[rank] // stride, n_l - 1)
        out["lo"].append(lo)
        out["hi"].append(hi)
        cf = cc = ivf = ivc = 0
        if l < L - 1 and lo <= hi:
            m = h.m[l]
            a, b = -(-lo // m), hi // m
            if a <= b:
                cf, cc = a, b - a + 1
            ivs = [i for i, (c, first, last) in enumerate(h.split(l).intervals) if lo <= first <= hi]
            ivf, ivc = (ivs[0], len(ivs)) if ivs else (0, 0)
        if l < L - 1:
            stride *= h.m[l]
        out["c_first"].append(cf)
        out["c_count"].append(cc)
        out["iv_first"].append(ivf)
        out["iv_count"].append(ivc)
    return out


@pytest.mark.parametrize("n_points,ms,k,workers", [(18, [3], 3, 6), (129, [4, 4], 3, 8),
                                                   (257, [16], 5, 4), (37, [3], 4, 5),
                                                   (16384, [128], 12, 8), (262145, [16], 8, 8)])
def test_rank_ranges_match_restatement(n_points, ms, k, workers):
    h = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, n_points), ms, k)
    lay = T.build_layout(h, workers)
    for r in range(workers):
        got = T.rank_ranges(h, workers, r)
        want = _ranges_reference(h, lay, r)
        for key in want:
            assert got[key] == want[key], (r, key)


def test_comm_groups_documented_decompositions():
    # test_runtime.cpp:75-109
    first, second = T.build_comm_groups(6, 3)
    assert first == [[0, 1, 2], [3, 4, 5]] and second == [[2, 3, 4]]
    first, second = T.build_comm_groups(6, 1)
    assert all(len(g) == 1 for g in first) and second == []


def _two_round_exchange(h, workers, k):
    """exchange_local_windows (parallel.cpp:134-194) simulated on sets."""
    lay = T.build_layout(h, workers)
    n = h.n_coarsest_points()
    first, second = T.build_comm_groups(n, k)
    owner = {p: r for r in range(workers) for p in range(lay.coarse_lo[r], lay.coarse_hi[r] + 1)}
    acc = [set(range(lay.coarse_lo[r], lay.coarse_hi[r] + 1)) for r in range(workers)]
    for decomposition, restrict in ((first, True), (second, False)):
        new = [set(a) for a in acc]
        for g in decomposition:
            owners = {owner[p] for p in g}
            if len(owners) < 2:
                continue
            for r in owners:
                for q in owners:
                    if q != r:
                        out = {p for p in acc[q] if p in g} if restrict else acc[q]
                        new[r] |= out
        acc = new
    result = []
    for r in range(workers):
        need = set()
        for p in range(lay.coarse_lo[r], lay.coarse_hi[r] + 1):
            need |= set(range(max(0, p - k + 1), p + 1))
        assert need <= acc[r], "two-round exchange must deliver every window index"
        result.append(need)
    return result


@pytest.mark.parametrize("n_points,m,k,workers", [(18, 3, 3, 6), (18, 3, 6, 6), (18, 3, 1, 6),
                                                  (37, 3, 4, 5), (257, 16, 5, 4),
                                                  (65, 4, 9, 8), (262145, 16, 8, 8)])
def test_direct_window_schedule_delivers_the_two_round_set(n_points, m, k, workers):
    h = T.build_hierarchy(T.TimeGrid.make(0.0, 1.0, n_points), [m], k)
    lay = T.build_layout(h, workers)
    want = _two_round_exchange(h, workers, k)
    for r in range(workers):
        have = set(range(lay.coarse_lo[r], lay.coarse_hi[r] + 1))
        for (src, first, count) in T.window_recvs(h, workers, r):
            assert src != r
            block = set(range(first, first + count))
            assert block <= set(range(lay.coarse_lo[src], lay.coarse_hi[src] + 1))
            have |= block
        assert want[r] <= have
        # nothing beyond the windows is moved
        assert have - set(range(lay.coarse_lo[r], lay.coarse_hi[r] + 1)) <= want[r]


def test_fullsize_fixtures_are_consistent():
    """tests/golden/fullsize_*.json (reference runs at BASELINE sizes): histories,
    iteration counts, failure cycles and sampled-row shapes agree."""
    import glob
    import json
    import os

    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    metas = sorted(glob.glob(os.path.join(gold, "fullsize_*.json")))
    assert metas
    for p in metas:
        meta = json.load(open(p))
        hist = meta["history"]
        if "failed_at_iteration" in meta:
            assert meta["code"] == 5 and len(hist) == meta["failed_at_iteration"] - 1
            continue
        assert meta["converged"] and meta["iterations"] == len(hist)
        assert hist[-1] <= meta["tol"] < min(hist[:-1])
        rows = np.load(p[:-5] + "_rows.npy")
        npts, n = {2: (4097, 127 * 127), 3: (16385, 4096), 4: (meta.get("n_points"), 511 * 511)}[meta["config"]]
        ds = meta.get("dof_stride", 1)
        assert rows.shape == (len(range(0, npts, meta["sample_every"])), len(range(0, n, ds)))
