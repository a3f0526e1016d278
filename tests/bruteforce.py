"""Independent brute-force definitions used to pin the oracle (tests only).

Nothing here is shared with oracle/ or the CUDA path.  Each helper restates a
definition from the paper / the DESIGN.md readings in the most direct
(non-recursive, O(N * nodes)) form, so that a mistake in the oracle's
recursive insertion / recursive walk shows up as a mismatch.
"""
from __future__ import annotations

import numpy as np

MAXLEVEL = 21


def prefix_nodes(keys_sorted: np.ndarray):
    """Brute-force octree topology from sorted 63-bit keys.

    PAPER.md:58-60 (§1): cubes are subdivided "until there is one particle per
    sub-cube"; reading L9 caps this at level 21 (buckets), L15 drops empty
    cells, L16 keeps single-child chains.  A node (l, prefix) exists iff at
    least one particle has that l-digit prefix and (l == 0 or the parent
    prefix holds >= 2 particles).  DFS pre-order with children in digit order
    equals lexicographic (first, level).  Returns [(level, first, count)].
    """
    keys = [int(k) for k in keys_sorted]
    n = len(keys)
    groups_by_level = []
    for lev in range(MAXLEVEL + 1):
        shift = 3 * (MAXLEVEL - lev)
        groups = {}
        for s, k in enumerate(keys):
            p = k >> shift
            if p not in groups:
                groups[p] = [s, 0]
            groups[p][1] += 1
        groups_by_level.append(groups)
    nodes = []
    for lev in range(MAXLEVEL + 1):
        for p, (first, count) in groups_by_level[lev].items():
            if lev == 0 or groups_by_level[lev - 1][p >> 3][1] >= 2:
                nodes.append((lev, first, count))
    nodes.sort(key=lambda t: (t[1], t[0]))
    assert nodes[0] == (0, 0, n)
    return nodes


def bh_bruteforce(mass, pos, keys_sorted, perm, L, theta, eps, G=1.0):
    """Non-recursive Barnes-Hut: node c contributes to target i iff c passes
    the interaction test and every proper ancestor of c is opened for i.

    PAPER.md:408-415 (§3): a remote cluster is treated as one body iff D > r/theta;
    readings L1-L5 (r = cell side L*2^-l, D to the centre of mass, strict, cells
    containing the target are always opened), L6 (Plummer softening).  Leaves
    interact directly; a bucket (level-21 cell with >= 2 particles) that is
    opened contributes its members j != i.
    Moments are flat sums over each node's particle range (no tree recursion).
    Returns (acc[N,3] with G, counts[N]) in user order.
    """
    mass = np.asarray(mass, np.float64)
    pos = np.asarray(pos, np.float64).reshape(-1, 3)
    n = mass.shape[0]
    perm = np.asarray(perm, np.int64)
    nodes = prefix_nodes(keys_sorted)
    rank = np.empty(n, np.int64)
    rank[perm] = np.arange(n)
    info = []
    for (lev, first, count) in nodes:
        members = perm[first:first + count]
        M = mass[members].sum()
        com = (mass[members, None] * pos[members]).sum(axis=0) / M
        info.append((lev, first, count, M, com))

    def is_ancestor(a, c):  # proper ancestor: a's range covers c's and a's level < c's level
        return a[1] <= c[1] and c[1] + c[2] <= a[1] + a[2] and a[0] < c[0]

    def mac(node, x):
        lev, _, _, _, com = node
        s = L * 2.0 ** (-lev)
        d = com - x
        d2 = d[0] * d[0]
        d2 = d2 + d[1] * d[1]
        d2 = d2 + d[2] * d[2]
        return s * s < theta * theta * d2

    acc = np.zeros((n, 3))
    cnt = np.zeros(n, np.int64)
    for i in range(n):
        x = pos[i]
        ki = rank[i]
        contrib = []
        opened = []
        for node in info:
            lev, first, count, M, com = node
            contains = first <= ki < first + count
            single = count == 1
            if single:
                opened.append(False)
            else:
                opened.append(contains or not mac(node, x))
        for c_idx, node in enumerate(info):
            lev, first, count, M, com = node
            ancestors_open = all(opened[a_idx] for a_idx, a in enumerate(info) if is_ancestor(a, node))
            if not ancestors_open:
                continue
            if count == 1:
                j = perm[first]
                if j != i:
                    contrib.append((mass[j], pos[j]))
            elif not opened[c_idx]:
                contrib.append((M, com))
            elif lev == MAXLEVEL:  # opened bucket: members
                for s in range(first, first + count):
                    j = perm[s]
                    if j != i:
                        contrib.append((mass[j], pos[j]))
        a = np.zeros(3)
        for m_s, x_s in contrib:
            d = x_s - x
            r2 = d @ d + eps * eps
            a += d * m_s / r2 ** 1.5
        acc[i] = G * a
        cnt[i] = len(contrib)
    return acc, cnt


def direct_numpy(mass, pos, eps, G=1.0, targets=None):
    """Softened O(N^2) direct sum with numpy (independent of oracle_direct)."""
    mass = np.asarray(mass, np.float64)
    pos = np.asarray(pos, np.float64).reshape(-1, 3)
    idx = np.arange(mass.shape[0]) if targets is None else np.asarray(targets)
    out = np.zeros((idx.shape[0], 3))
    for t, i in enumerate(idx):
        d = pos - pos[i]
        r2 = (d * d).sum(axis=1) + eps * eps
        r2[i] = np.inf
        w = mass / (r2 * np.sqrt(r2))
        out[t] = G * (d * w[:, None]).sum(axis=0)
    return out


def decode_key(k: int):
    """Inverse of the x-major 3-bit interleave (bit 3b+2 <- x bit b)."""
    qx = qy = qz = 0
    for b in range(MAXLEVEL):
        qx |= ((k >> (3 * b + 2)) & 1) << b
        qy |= ((k >> (3 * b + 1)) & 1) << b
        qz |= ((k >> (3 * b)) & 1) << b
    return qx, qy, qz


def decode_keys_np(keys: np.ndarray):
    keys = np.asarray(keys, np.uint64)
    q = np.zeros((keys.shape[0], 3), np.uint64)
    for b in range(MAXLEVEL):
        for a, off in enumerate((2, 1, 0)):
            q[:, a] |= ((keys >> np.uint64(3 * b + off)) & np.uint64(1)) << np.uint64(b)
    return q
