"""Oracle: adaptive octree from Morton codes and the KIFMM interaction lists.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product path.

PAPER.md Sec. 2.2 (line 135): "Generation of an octree partitioning of the domain
into boxes", and (line 143) "At the finest level of the tree, the complete
integrals are computed by adding the contributions of points in the near zone
using direct summation".  The paper delegates the tree and the lists to the
KIFMM of its refs [kifmm, pvfmm]; the definitions below are the standard adaptive
KIFMM ones, stated here as reading R5:

  root cube     lo/hi = componentwise min/max over sources U targets (fp64),
                side = max_a(hi_a - lo_a) * (1 + 2**-10)  (1.0 if that is 0),
                origin_a = (lo_a + hi_a)/2 - side/2.
  Morton key    q_a = floor((x_a - origin_a) * (2**20 / side)), clamped to [0, 2**20 - 1],
                every operation one IEEE fp64 op (no fused multiply-add);
                key = interleave(q_x, q_y, q_z), x the most significant bit of each
                triple, so the child octant is c = 4 bx + 2 by + bz.
  point order   stable sort of (sources, then targets) by key.
  refinement    a box at level l < 20 is split iff max(n_src, n_trg) > max_pts;
                only non-empty children are created.
  box order     level by level; inside a level by Morton key (= parent order, then octant).
  adjacency     two boxes are adjacent iff their closed cubes intersect and neither
                contains the other.
  colleagues(B) same-level boxes at Chebyshev anchor distance <= 1 (B included).
  U(B), B leaf  leaves adjacent to B, and B itself.
  V(B)          children of colleagues of parent(B) that are not adjacent to B.
  W(B), B leaf  descendants A of colleagues of B with A not adjacent to B and
                parent(A) adjacent to B.
  X(B)          { A : B in W(A) }.

Coverage (pinned in tests/test_oracle_tree.py): for every target leaf B and source
leaf A, exactly one of  A in U(B);  A' in V(B') for ancestors-or-self A', B';
A' in W(B) for an ancestor-or-self A';  A in X(B') for an ancestor-or-self B'.
"""
from __future__ import annotations

import numpy as np

MAXLEVEL = 20
PAD = 1.0 + 2.0 ** -10


def root_cube(points: np.ndarray):
    """(origin[3], side) of the root cube, reading R5."""
    p = np.asarray(points, np.float64).reshape(-1, 3)
    lo = p.min(axis=0)
    hi = p.max(axis=0)
    side = float(np.max(hi - lo))
    side = 1.0 if side == 0.0 else side * PAD
    origin = (lo + hi) * 0.5 - side * 0.5
    return origin, side


def quantize(points: np.ndarray, origin, side):
    """integer grid coordinates at level MAXLEVEL (one fp64 op per step, as in reading R5)."""
    p = np.asarray(points, np.float64).reshape(-1, 3)
    scale = float(2 ** MAXLEVEL) / side
    t = (p - origin[None, :]) * scale
    q = np.floor(t)
    q = np.clip(q, 0, 2 ** MAXLEVEL - 1).astype(np.int64)
    return q


def morton(q: np.ndarray) -> np.ndarray:
    """interleave the 20 bits of qx, qy, qz: bit b of qx -> bit 3b+2, qy -> 3b+1, qz -> 3b."""
    q = np.asarray(q, np.int64)
    key = np.zeros(q.shape[0], np.int64)
    for b in range(MAXLEVEL):
        key |= ((q[:, 0] >> b) & 1) << (3 * b + 2)
        key |= ((q[:, 1] >> b) & 1) << (3 * b + 1)
        key |= ((q[:, 2] >> b) & 1) << (3 * b)
    return key


class Tree:
    """flat arrays over boxes (box id = position in level-then-Morton order)."""

    def __init__(self):
        self.level = None      # (nb,)
        self.anchor = None     # (nb, 3) integer anchor at its own level
        self.parent = None     # (nb,)   -1 for the root
        self.child = None      # (nb, 8) -1 where absent
        self.begin = None      # (nb,)   range in the sorted point array
        self.end = None
        self.src_begin = None  # range in the sorted source array
        self.src_end = None
        self.trg_begin = None  # range in the sorted target array
        self.trg_end = None
        self.leaf = None       # (nb,) bool
        self.origin = None
        self.side = None
        self.keys = None       # sorted keys of all points
        self.perm = None       # sorted position -> original point index (sources first)
        self.src_perm = None   # sorted-source position -> original source index
        self.trg_perm = None
        self.level_start = None

    @property
    def nboxes(self):
        return self.level.shape[0]

    def center(self, b):
        h = self.side / 2.0 ** self.level[b]
        return self.origin + (self.anchor[b] + 0.5) * h

    def half_width(self, b):
        return self.side / 2.0 ** (self.level[b] + 1)


def build_tree(src: np.ndarray, trg: np.ndarray, max_pts: int) -> Tree:
    src = np.asarray(src, np.float64).reshape(-1, 3)
    trg = np.asarray(trg, np.float64).reshape(-1, 3)
    ns, nt = src.shape[0], trg.shape[0]
    pts = np.concatenate([src, trg])
    is_src = np.concatenate([np.ones(ns, bool), np.zeros(nt, bool)])
    origin, side = root_cube(pts)
    keys = morton(quantize(pts, origin, side))
    perm = np.argsort(keys, kind="stable")
    skeys = keys[perm]
    sis = is_src[perm]
    csrc = np.concatenate([[0], np.cumsum(sis)])            # sources before sorted position i
    ctrg = np.concatenate([[0], np.cumsum(~sis)])

    level, anchor, parent, begin, end, leaf = [0], [(0, 0, 0)], [-1], [0], [ns + nt], []
    child = []
    cur = [0]
    lvl = 0
    while cur:
        nxt = []
        for b in cur:
            nsb = csrc[end[b]] - csrc[begin[b]]
            ntb = ctrg[end[b]] - ctrg[begin[b]]
            ch = [-1] * 8
            if lvl < MAXLEVEL and max(nsb, ntb) > max_pts:
                shift = 3 * (MAXLEVEL - lvl - 1)
                a = anchor[b]
                prefix = 0
                for bit in range(lvl):   # parent key prefix from the anchor
                    s = lvl - 1 - bit
                    prefix = (prefix << 3) | (((a[0] >> s) & 1) << 2) | (((a[1] >> s) & 1) << 1) | ((a[2] >> s) & 1)
                for c in range(8):
                    lo_key = ((prefix << 3) | c) << shift
                    hi_key = ((prefix << 3) + c + 1) << shift
                    i0 = int(np.searchsorted(skeys, lo_key, side="left"))
                    i1 = int(np.searchsorted(skeys, hi_key, side="left"))
                    i0 = max(i0, begin[b])
                    i1 = min(i1, end[b])
                    if i1 > i0:
                        ch[c] = len(level)
                        level.append(lvl + 1)
                        anchor.append((2 * a[0] + (c >> 2), 2 * a[1] + ((c >> 1) & 1), 2 * a[2] + (c & 1)))
                        parent.append(b)
                        begin.append(i0)
                        end.append(i1)
                        nxt.append(ch[c])
            child.append(ch)
        cur = nxt
        lvl += 1
    T = Tree()
    T.level = np.array(level, np.int64)
    T.anchor = np.array(anchor, np.int64)
    T.parent = np.array(parent, np.int64)
    T.child = np.array(child, np.int64)
    T.begin = np.array(begin, np.int64)
    T.end = np.array(end, np.int64)
    T.leaf = np.all(T.child < 0, axis=1)
    T.src_begin = csrc[T.begin]
    T.src_end = csrc[T.end]
    T.trg_begin = ctrg[T.begin]
    T.trg_end = ctrg[T.end]
    T.origin, T.side = origin, side
    T.keys = skeys
    T.perm = perm
    T.src_perm = perm[sis]
    T.trg_perm = perm[~sis] - ns
    T.level_start = np.searchsorted(T.level, np.arange(T.level.max() + 2))
    return T


def box_key(T: Tree, b: int) -> int:
    """Morton key of a box = interleaved anchor bits at its level (identifies a box
    independently of any numbering)."""
    a = T.anchor[b]
    key = 0
    for s in range(T.level[b] - 1, -1, -1):
        key = (key << 3) | (((a[0] >> s) & 1) << 2) | (((a[1] >> s) & 1) << 1) | ((a[2] >> s) & 1)
    return key


def _extent(T, b, L):
    """closed integer interval [lo, hi] of box b in level-L units."""
    sc = 1 << (L - T.level[b])
    lo = T.anchor[b] * sc
    return lo, lo + sc


def adjacent(T: Tree, a: int, b: int) -> bool:
    """closed cubes intersect and neither contains the other (reading R5)."""
    L = max(T.level[a], T.level[b])
    alo, ahi = _extent(T, a, L)
    blo, bhi = _extent(T, b, L)
    touch = np.all(alo <= bhi) and np.all(blo <= ahi)
    if not touch:
        return False
    a_in_b = np.all(alo >= blo) and np.all(ahi <= bhi)
    b_in_a = np.all(blo >= alo) and np.all(bhi <= ahi)
    return not (a_in_b or b_in_a)


def colleagues(T: Tree, b: int, index=None):
    """same-level boxes within Chebyshev anchor distance 1 (b included), ascending id."""
    if index is None:
        index = level_index(T)
    l = int(T.level[b])
    a = T.anchor[b]
    out = []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                k = (l, a[0] + dx, a[1] + dy, a[2] + dz)
                if k in index:
                    out.append(index[k])
    return sorted(out)


def level_index(T: Tree):
    return {(int(T.level[b]), int(T.anchor[b, 0]), int(T.anchor[b, 1]), int(T.anchor[b, 2])): b
            for b in range(T.nboxes)}


def build_lists(T: Tree):
    """U, V, W, X lists by the definitions of reading R5, computed box by box.
    Returns dict name -> list (per box) of ascending box ids ([] where undefined)."""
    nb = T.nboxes
    index = level_index(T)
    coll = [colleagues(T, b, index) for b in range(nb)]
    U = [[] for _ in range(nb)]
    V = [[] for _ in range(nb)]
    W = [[] for _ in range(nb)]
    X = [[] for _ in range(nb)]
    for b in range(nb):
        p = T.parent[b]
        if p >= 0:
            for c in coll[p]:
                for a in T.child[c]:
                    if a >= 0 and np.max(np.abs(T.anchor[a] - T.anchor[b])) > 1:
                        V[b].append(int(a))
        if not T.leaf[b]:
            continue
        # same-level adjacent leaves (and b itself)
        for c in coll[b]:
            if T.leaf[c]:
                U[b].append(c)
        # descend into non-leaf colleagues: adjacent leaves -> U, first non-adjacent -> W
        stack = [int(a) for c in coll[b] if c != b and not T.leaf[c] for a in T.child[c] if a >= 0]
        while stack:
            a = stack.pop()
            if adjacent(T, a, b):
                if T.leaf[a]:
                    U[b].append(a)
                else:
                    stack.extend(int(x) for x in T.child[a] if x >= 0)
            else:
                W[b].append(a)
    # coarser adjacent leaves are the dual of finer adjacent leaves; X is the dual of W
    for b in range(nb):
        for a in list(U[b]):
            if T.level[a] > T.level[b]:
                U[a].append(b)
        for a in W[b]:
            X[a].append(b)
    return {k: [sorted(set(v)) for v in L] for k, L in (("U", U), ("V", V), ("W", W), ("X", X))}


def build_lists_bruteforce(T: Tree):
    """the same definitions evaluated over all box pairs (O(nb^2); tiny trees only)."""
    nb = T.nboxes
    U = [[] for _ in range(nb)]
    V = [[] for _ in range(nb)]
    W = [[] for _ in range(nb)]
    X = [[] for _ in range(nb)]

    def is_colleague(a, b):
        return T.level[a] == T.level[b] and np.max(np.abs(T.anchor[a] - T.anchor[b])) <= 1

    def is_desc(a, c):          # a strict descendant of c
        while T.parent[a] >= 0:
            a = T.parent[a]
            if a == c:
                return True
        return False

    for b in range(nb):
        for a in range(nb):
            if T.parent[b] >= 0 and T.parent[a] >= 0 and is_colleague(T.parent[a], T.parent[b]) \
                    and T.level[a] == T.level[b] and not is_colleague(a, b):
                V[b].append(a)
            if T.leaf[b] and T.leaf[a] and (a == b or adjacent(T, a, b)):
                U[b].append(a)
            if T.leaf[b] and T.level[a] > T.level[b] and not adjacent(T, a, b) \
                    and adjacent(T, T.parent[a], b) \
                    and any(is_desc(a, c) for c in range(nb) if is_colleague(c, b)):
                W[b].append(a)
    for b in range(nb):
        for a in W[b]:
            X[a].append(b)
    return {k: [sorted(v) for v in L] for k, L in (("U", U), ("V", V), ("W", W), ("X", X))}
