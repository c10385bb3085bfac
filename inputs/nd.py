"""Geometric nested dissection on structured grids (host preprocessing).

Stand-in for the paper's compressed-graph METIS nested dissection (Sec. 3.3,
PAPER.md:988-1046; METIS is not in the container).  Recursive bisection of the
box along its longest axis with a one-plane separator; each leaf (<= `leaf`
nodes) and each separator is ordered lexicographically (x fastest) and cut into
initial blocks of up to `block` consecutive unknowns (stand-in for the ILU(1,tau)
block guess of Sec. 3.4, which is NEXT-3 in SURVEY.md 8(f)).
Children are ordered before their separator, left before right (postorder).
"""
from __future__ import annotations

import numpy as np


def _lex_nodes(x0, x1, y0, y1, z0, z1, nx, ny):
    xs = np.arange(x0, x1)
    ys = np.arange(y0, y1)
    zs = np.arange(z0, z1)
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    return (X + nx * (Y + ny * Z)).ravel()


def _cut(count, block):
    out = []
    while count > 0:
        b = min(block, count)
        out.append(b)
        count -= b
    return out


def grid_nd(nx, ny, nz, leaf=512, block=8, top_levels=0):
    """Return (perm, block_sizes, block_part).

    perm[i] = original index of the unknown placed at position i (Ã = A(perm, perm)).
    block_part[K] = top-level subtree id (0..2^top_levels-1) of block K, or -1 for
    blocks of the top `top_levels` separators (used for multi-GPU partitioning).
    """
    perm_parts, sizes, parts = [], [], []
    counter = [0]

    def rec(box, depth, part):
        x0, x1, y0, y1, z0, z1 = box
        dims = [x1 - x0, y1 - y0, z1 - z0]
        cnt = dims[0] * dims[1] * dims[2]
        if cnt == 0:
            return
        if depth == top_levels and top_levels > 0 and part < 0:
            part = counter[0]
            counter[0] += 1
        if cnt <= leaf or max(dims) < 3:
            if top_levels > 0 and part < 0:      # a leaf above the top levels is a subtree of its own
                part = counter[0]
                counter[0] += 1
            nodes = _lex_nodes(x0, x1, y0, y1, z0, z1, nx, ny)
            perm_parts.append(nodes)
            bs = _cut(len(nodes), block)
            sizes.extend(bs)
            parts.extend([part] * len(bs))
            return
        ax = int(np.argmax(dims))
        lo = [x0, y0, z0][ax]
        hi = [x1, y1, z1][ax]
        mid = (lo + hi) // 2
        left = list(box)
        right = list(box)
        sep = list(box)
        left[2 * ax + 1] = mid
        right[2 * ax] = mid + 1
        sep[2 * ax] = mid
        sep[2 * ax + 1] = mid + 1
        rec(tuple(left), depth + 1, part)
        rec(tuple(right), depth + 1, part)
        nodes = _lex_nodes(*sep, nx, ny)
        perm_parts.append(nodes)
        bs = _cut(len(nodes), block)
        sizes.extend(bs)
        parts.extend([part] * len(bs))

    rec((0, nx, 0, ny, 0, nz), 0, -1)
    perm = np.concatenate(perm_parts).astype(np.int64)
    assert len(perm) == nx * ny * nz
    return perm, np.asarray(sizes, dtype=np.int32), np.asarray(parts, dtype=np.int32)


def expand_dof(perm, sizes, parts, dof):
    """Nodal ordering/blocking -> unknown ordering (dof unknowns per node, nodal blocks)."""
    perm = np.asarray(perm, dtype=np.int64)
    p = (perm[:, None] * dof + np.arange(dof)[None, :]).ravel()
    return p, np.asarray(sizes, dtype=np.int32) * dof, parts
