"""Marching-cubes triangulation table, generated.

The reference extracts meshes with scikit-image's 256-case marching cubes
(`measure.marching_cubes(method="lorensen")`, gs/mesher.py:136-146), which is
not available here.  This module derives an equivalent 256-case table from the
cube topology instead of transcribing one: for every corner sign pattern the
edge crossings on each face are joined into segments, the segments close into
loops, and each loop is fan-triangulated.  On a face whose diagonal corners
share a sign (the ambiguous case) the segments separate the *inside*
corners; the rule depends only on that face's four signs, so the two cells
sharing a face always agree and the surface is watertight.

Conventions (shared with csrc/gsb_mesh.cu):
  corner k = 4 dx + 2 dy + dz (x-major, like the grid corners)
  edge e = 4 axis + j, j enumerating the other two coordinates (lo-hi order)
  a corner is inside when value < level; triangles are oriented with their
  normal pointing from inside to outside.
"""

from __future__ import annotations

import numpy as np

CORNERS = np.array([[(k >> 2) & 1, (k >> 1) & 1, k & 1] for k in range(8)], dtype=np.int64)


def _edges():
    e = []
    for axis in range(3):
        others = [a for a in range(3) if a != axis]
        for j in range(4):
            c = [0, 0, 0]
            c[others[0]] = (j >> 1) & 1
            c[others[1]] = j & 1
            lo = c.copy()
            hi = c.copy()
            hi[axis] = 1
            e.append((4 * lo[0] + 2 * lo[1] + lo[2], 4 * hi[0] + 2 * hi[1] + hi[2]))
    return e


EDGES = _edges()  # 12 (corner_a, corner_b), a < b along the edge axis


def _faces():
    """Each face: its 4 corners in cyclic order and the 4 edges between them."""
    faces = []
    for axis in range(3):
        u, v = [a for a in range(3) if a != axis]
        for side in (0, 1):
            cyc = []
            for du, dv in ((0, 0), (1, 0), (1, 1), (0, 1)):
                c = [0, 0, 0]
                c[axis], c[u], c[v] = side, du, dv
                cyc.append(4 * c[0] + 2 * c[1] + c[2])
            ed = []
            for i in range(4):
                a, b = cyc[i], cyc[(i + 1) % 4]
                ed.append(next(k for k, (p, q) in enumerate(EDGES) if {p, q} == {a, b}))
            faces.append((cyc, ed))
    return faces


FACES = _faces()


def _case(mask):
    inside = [(mask >> k) & 1 for k in range(8)]
    cut = [k for k, (a, b) in enumerate(EDGES) if inside[a] != inside[b]]
    if not cut:
        return []
    nbr = {e: [] for e in cut}
    for cyc, ed in FACES:
        s = [inside[c] for c in cyc]
        cuts = [i for i in range(4) if s[i] != s[(i + 1) % 4]]  # edge i joins corners i, i+1
        if len(cuts) == 2:
            pairs = [(cuts[0], cuts[1])]
        elif len(cuts) == 4:
            # ambiguous face: separate the inside corners, i.e. cut off each
            # inside corner with the segment joining its two incident edges
            pairs = []
            for i in range(4):
                if s[i]:
                    pairs.append(((i - 1) % 4, i))
        else:
            pairs = []
        for i, j in pairs:
            nbr[ed[i]].append(ed[j])
            nbr[ed[j]].append(ed[i])
    # loops
    seen, loops = set(), []
    for e0 in cut:
        if e0 in seen:
            continue
        loop, prev, cur = [e0], None, e0
        seen.add(e0)
        while True:
            nx = [x for x in nbr[cur] if x != prev]
            nxt = nx[0] if nx else None
            if nxt is None or nxt == e0:
                break
            loop.append(nxt)
            seen.add(nxt)
            prev, cur = cur, nxt
        loops.append(loop)
    tris = []
    for loop in loops:
        mid = np.array([(CORNERS[EDGES[e][0]] + CORNERS[EDGES[e][1]]) / 2.0 for e in loop])
        out_dir = np.zeros(3)  # average inside -> outside direction along the cut edges
        for e in loop:
            a, b = EDGES[e]
            out_dir += (CORNERS[b] - CORNERS[a]) * (1.0 if inside[a] else -1.0)
        n = np.zeros(3)  # Newell normal of the loop
        for i in range(len(loop)):
            p, q = mid[i], mid[(i + 1) % len(loop)]
            n += np.cross(p, q)
        if np.dot(n, out_dir) < 0:
            loop = loop[::-1]
        for i in range(1, len(loop) - 1):
            tris.append((loop[0], loop[i], loop[i + 1]))
    return tris


def build():
    cases = [_case(m) for m in range(256)]
    max_t = max(len(t) for t in cases)
    tab = -np.ones((256, 3 * max_t + 1), dtype=np.int8)
    ntri = np.zeros(256, dtype=np.int8)
    for m, t in enumerate(cases):
        ntri[m] = len(t)
        for i, tri in enumerate(t):
            tab[m, 3 * i:3 * i + 3] = tri
    return tab, ntri, max_t


TABLE, NTRI, MAX_TRI = build()
EDGE_CORNERS = np.array(EDGES, dtype=np.int8)  # (12, 2)
