"""Pins for oracle/tree.py: Morton codes by hand, partition invariants, the lists
against a brute-force evaluation of their definitions, and the FMM coverage
property (every source-leaf/target-leaf pair accounted for exactly once)."""
import numpy as np
import pytest

from oracle import tree as T
from workloads import geometry


def test_morton_hand_values():
    q = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 1], [2, 0, 0], [1, 1, 1],
                  [2 ** 19, 0, 0], [3, 5, 6], [2 ** 20 - 1] * 3])
    k = T.morton(q)
    # (3,5,6): bit0 (1,1,0)->0b110, bit1 (1,0,1)->0b101, bit2 (0,1,1)->0b011
    expect = [4, 2, 1, 32, 7, 1 << 59, 0b011_101_110, 2 ** 60 - 1]
    assert list(k) == expect


def test_quantize_extremes_inside():
    rng = np.random.default_rng(0)
    p = rng.uniform(-3, 5, (1000, 3))
    o, s = T.root_cube(p)
    q = T.quantize(p, o, s)
    assert q.min() >= 0 and q.max() <= 2 ** 20 - 1
    # the padded cube strictly contains the extreme points (no clamping needed)
    t = (p - o) * (2 ** 20 / s)
    assert t.min() > 0 and t.max() < 2 ** 20


def _clouds():
    rng = np.random.default_rng(7)
    uni = rng.uniform(0, 1, (600, 3))
    clus = np.concatenate([rng.normal(0.2, 0.01, (300, 3)), rng.uniform(0, 1, (200, 3))])
    sph = geometry.sphere_points(700, seed=3)
    return [("uniform", uni, uni, 16), ("cluster", clus, clus, 8), ("sphere", sph, sph, 12),
            ("split", uni[:300], sph[:400] * 0.4 + 0.5, 10)]


@pytest.mark.parametrize("name,src,trg,s", _clouds())
def test_tree_partition_invariants(name, src, trg, s):
    tr = T.build_tree(src, trg, s)
    leaves = np.nonzero(tr.leaf)[0]
    # leaf point ranges partition [0, N)
    rng_ = sorted((tr.begin[b], tr.end[b]) for b in leaves)
    assert rng_[0][0] == 0 and rng_[-1][1] == src.shape[0] + trg.shape[0]
    assert all(a[1] == b[0] for a, b in zip(rng_, rng_[1:]))
    # refinement criterion
    ns = tr.src_end - tr.src_begin
    nt = tr.trg_end - tr.trg_begin
    assert np.all(np.maximum(ns, nt)[leaves] <= s) or tr.level.max() == T.MAXLEVEL
    inner = np.nonzero(~tr.leaf)[0]
    assert np.all(np.maximum(ns, nt)[inner] > s)
    # every point lies geometrically inside its leaf cube
    pts = np.concatenate([src, trg])
    for b in leaves:
        c, h = tr.center(b), tr.half_width(b)
        p = pts[tr.perm[tr.begin[b]:tr.end[b]]]
        assert np.all(np.abs(p - c) <= h * (1 + 1e-12))
    # box keys ascend within each level
    for l in range(tr.level.max() + 1):
        ks = [T.box_key(tr, b) for b in np.nonzero(tr.level == l)[0]]
        assert ks == sorted(ks) and len(set(ks)) == len(ks)


@pytest.mark.parametrize("name,src,trg,s", _clouds())
def test_lists_match_bruteforce_definition(name, src, trg, s):
    tr = T.build_tree(src, trg, s)
    a = T.build_lists(tr)
    b = T.build_lists_bruteforce(tr)
    for k in "UVWX":
        assert a[k] == b[k], k


@pytest.mark.parametrize("name,src,trg,s", _clouds())
def test_lists_cover_every_pair_exactly_once(name, src, trg, s):
    tr = T.build_tree(src, trg, s)
    L = T.build_lists(tr)
    sets = {k: [set(v) for v in L[k]] for k in "UVWX"}

    def anc(b):
        out = [b]
        while tr.parent[out[-1]] >= 0:
            out.append(int(tr.parent[out[-1]]))
        return out

    leaves = np.nonzero(tr.leaf)[0]
    for B in leaves:
        aB = anc(B)
        for A in leaves:
            aA = anc(A)
            n = int(A in sets["U"][B])
            n += sum(1 for b2 in aB for a2 in aA if a2 in sets["V"][b2])
            n += sum(1 for a2 in aA if a2 in sets["W"][B])
            n += sum(1 for b2 in aB if A in sets["X"][b2])
            assert n == 1, (B, A, n)


def test_separation_of_far_lists():
    src = geometry.sphere_points(900, seed=11)
    tr = T.build_tree(src, src, 10)
    L = T.build_lists(tr)
    for b in range(tr.nboxes):
        for a in L["V"][b]:
            assert tr.level[a] == tr.level[b]
            assert np.max(np.abs(tr.anchor[a] - tr.anchor[b])) >= 2
        for a in L["W"][b]:
            assert tr.level[a] > tr.level[b] and not T.adjacent(tr, a, b)
        for a in L["U"][b]:
            assert tr.leaf[a] and (a == b or T.adjacent(tr, a, b))
