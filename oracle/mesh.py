"""Marching cubes on the phi field, written out plainly (oracle side of NEXT-4).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py): used by tests/ to check the
CUDA path's pf_mesh; shares no code (and no tables) with it.

PAPER.md:246-251 (§Input/Output): "a custom marching cubes algorithm based on
[lorensen1987marching] ... generates meshes locally on each block, using the
phi values as input.  For each phase, a mesh is generated, describing the
interface between this phase and all other phases.  The marching cubes
algorithm extends to the ghost regions such that the local meshes can be
stitched together".  The paper gives no case table; DESIGN.md §3 reading R26
fixes the variant both sides implement:

  * samples at cell centres; cube (i, j, k) has corners (i+dx, j+dy, k+dz),
    dx, dy, dz in {0, 1}, corner number dx + 2 dy + 4 dz; periodic in x and y,
    cubes k = 0 .. NZ-2 only in z (no cube reaches into the zero-flux ghost);
  * a corner is inside when phi_a > iso (iso = 1/2);
  * cube edges 0-3 run along x at (dy, dz) = (e & 1, e >> 1), 4-7 along y at
    (dx, dz), 8-11 along z at (dx, dy); an edge crosses when its two corners
    differ in insideness; its vertex lies at t = (iso - f0) / (f1 - f0) from
    the lower corner, position ((index + 0.5) + t) * dx on its axis and
    (index + 0.5) * dx on the others, z index counted from the window origin;
    x, y indices wrapped into [0, N);
  * the surface inside a cube is assembled face by face: on each cube face,
    corners in counter-clockwise order seen from outside, every maximal run of
    consecutive inside corners q_a..q_b contributes one directed segment from
    its entry edge (q_a-1, q_a) to its exit edge (q_b, q_b+1).  Diagonal faces
    therefore separate the two inside corners; the rule sees only the face's
    own corners, so the two cubes sharing a face agree and the mesh is
    watertight;
  * the segments close into cycles (of 3 to 7 edges); each cycle is rotated
    to start at its apex v0 and fanned into triangles (v0, v_t, v_t+1).  The
    apex is the smallest cube-local edge number in the cycle that shares no
    cube face with any non-adjacent cycle vertex, so that no fan diagonal
    lies in a cube face (a cycle crossing an ambiguous face twice would
    otherwise put a chord into the face the neighbour cube also meshes; such
    an apex exists for every cycle of the 256 cases, checked exhaustively in
    P16).  Cycles in order of their smallest edge.  With this
    segment direction the triangles' right-hand normals point out of the
    phase, down the gradient of phi_a;
  * a vertex is identified by its global grid edge: id = 3 (i + NX (j + NY k))
    + axis with (i, j, k) the edge's lower corner (wrapped).

Pinned in tests/test_oracle_pins.py (P16): empty mesh for a uniform field,
exact area of a plane, a sphere's area / volume / Euler characteristic,
watertight + consistently oriented meshes of random fields, normals pointing
down the gradient.
"""
from __future__ import annotations

import numpy as np

# cube edges: (corner0, corner1, axis); corner0 is the lower end
EDGES = []
for e in range(4):
    dy, dz = e & 1, e >> 1
    EDGES.append((2 * dy + 4 * dz, 1 + 2 * dy + 4 * dz, 0))
for e in range(4):
    dx, dz = e & 1, e >> 1
    EDGES.append((dx + 4 * dz, dx + 2 + 4 * dz, 1))
for e in range(4):
    dx, dy = e & 1, e >> 1
    EDGES.append((dx + 2 * dy, dx + 2 * dy + 4, 2))


def _corner(dx, dy, dz):
    return dx + 2 * dy + 4 * dz


def _faces():
    """Six faces, corners counter-clockwise seen from outside (right-handed
    about the outward normal)."""
    faces = []
    for a in range(3):
        u, v = (a + 1) % 3, (a + 2) % 3        # u x v = +e_a
        for side in (0, 1):
            uv = [(0, 0), (1, 0), (1, 1), (0, 1)]
            if side == 0:
                uv = uv[::-1]                    # outward normal -e_a: reverse
            cs = []
            for (pu, pv) in uv:
                d = [0, 0, 0]
                d[a], d[u], d[v] = side, pu, pv
                cs.append(_corner(*d))
            faces.append(cs)
    return faces


FACES = _faces()


def _edge_of(c0, c1):
    for e, (a, b, _) in enumerate(EDGES):
        if {a, b} == {c0, c1}:
            return e
    raise AssertionError


def _share_face(e0, e1):
    a = set(EDGES[e0][:2]) | set(EDGES[e1][:2])
    return any(a <= set(cs) for cs in FACES)


def cube_triangles(inside):
    """inside[8] (bools) -> list of triangles of cube-local edge numbers."""
    nxt = {}
    for cs in FACES:
        ins = [inside[c] for c in cs]
        if all(ins) or not any(ins):
            continue
        for a in range(4):
            if ins[a] and not ins[(a - 1) % 4]:          # a run starts at q_a
                b = a
                while ins[(b + 1) % 4]:
                    b = (b + 1) % 4
                exit_e = _edge_of(cs[b], cs[(b + 1) % 4])
                entry_e = _edge_of(cs[(a - 1) % 4], cs[a])
                assert entry_e not in nxt
                nxt[entry_e] = exit_e
    tris = []
    seen = set()
    for start in sorted(nxt):
        if start in seen:
            continue
        cyc = [start]
        seen.add(start)
        e = nxt[start]
        while e != start:
            cyc.append(e)
            seen.add(e)
            e = nxt[e]
        m = len(cyc)
        r = min((r for r in range(m)
                 if not any(_share_face(cyc[r], cyc[(r + t) % m]) for t in range(2, m - 1))),
                key=lambda r: cyc[r])
        cyc = cyc[r:] + cyc[:r]
        for t in range(1, m - 1):
            tris.append((cyc[0], cyc[t], cyc[t + 1]))
    return tris


def marching_cubes(phi_a, iso=0.5, dx=1.0, z_origin=0, cubes=None):
    """phi_a[NZ, NY, NX] (float64, the interior of one phase) -> (edge ids
    int64[T, 3], vertex positions float64[T, 3, 3] as (x, y, z)).  `cubes`
    optionally restricts to a list of (i, j, k) lower corners (sampling)."""
    phi_a = np.asarray(phi_a, dtype=np.float64)
    NZ, NY, NX = phi_a.shape
    if cubes is None:
        # classification only narrows the loop; every candidate is walked below
        ins = phi_a > iso
        nb = [np.roll(np.roll(ins[dz:NZ - 1 + dz], -dy, axis=1), -dx, axis=2)
              for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)]
        mixed = np.any(np.stack(nb) != nb[0], axis=0)
        cubes = [(int(i), int(j), int(k)) for k, j, i in np.argwhere(mixed)]
        cubes.sort(key=lambda c: (c[2], c[1], c[0]))
    ids, pos = [], []
    for (i, j, k) in cubes:
        f = [0.0] * 8
        for c in range(8):
            cx, cy, cz = c & 1, (c >> 1) & 1, c >> 2
            f[c] = float(phi_a[k + cz, (j + cy) % NY, (i + cx) % NX])
        tris = cube_triangles([v > iso for v in f])
        for tri in tris:
            tid, tpos = [], []
            for e in tri:
                c0, c1, ax = EDGES[e]
                lo = [(i + (c0 & 1)) % NX, (j + ((c0 >> 1) & 1)) % NY, k + (c0 >> 2)]
                t = (iso - f[c0]) / (f[c1] - f[c0])
                tid.append(3 * (lo[0] + NX * (lo[1] + NY * lo[2])) + ax)
                g = [lo[0], lo[1], lo[2] + z_origin]
                p = [(g[q] + 0.5) * dx for q in range(3)]
                p[ax] = ((g[ax] + 0.5) + t) * dx
                tpos.append(p)
            ids.append(tid)
            pos.append(tpos)
    return np.array(ids, dtype=np.int64).reshape(-1, 3), np.array(pos, dtype=np.float64).reshape(-1, 3, 3)


def canonical(ids):
    """Rotate each triangle to start at its smallest id (orientation kept)
    and sort the list: a representation independent of emission order."""
    ids = np.asarray(ids, dtype=np.int64).reshape(-1, 3)
    if len(ids) == 0:
        return ids
    r = np.argmin(ids, axis=1)
    rot = np.stack([ids[np.arange(len(ids)), (r + s) % 3] for s in range(3)], axis=1)
    return rot[np.lexsort(rot.T[::-1])]
