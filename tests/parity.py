"""Parity comparison between the CUDA factors and the oracle's (test helper).

SURVEY.md 8(c) reading 14: "relative 1e-10" is checked normwise per stored
object: each L row, each Ũ column and each D block,
    max|g - o| <= tol * max|o|   (over that row / column / block).
Patterns must be identical (near-threshold decisions are replayed in the oracle
before comparing, reading 15).
"""
from __future__ import annotations

import numpy as np


def compare_factors(g, o, tol=1e-10):
    """Return a dict of discrepancies (empty problems list == parity)."""
    problems = []
    if g.nblk != o.nblk or not np.array_equal(np.asarray(g.bstart), np.asarray(o.bstart)):
        problems.append("partition differs: %d vs %d blocks" % (g.nblk, o.nblk))
        return {"problems": problems, "max_rel": np.inf}
    worst = 0.0
    for K in range(o.nblk):
        s, e, gr, gL, gc, gU, gD = g.block(K)
        _, _, orr, oL, oc, oU, oD = o.block(K)
        if not np.array_equal(gr, orr):
            problems.append("block %d: L row pattern differs (%d vs %d rows)" % (K, len(gr), len(orr)))
            continue
        if not np.array_equal(gc, oc):
            problems.append("block %d: U col pattern differs (%d vs %d cols)" % (K, len(gc), len(oc)))
            continue
        for a, b_ in ((gL, oL), (gU.T, oU.T)):
            if a.size:
                den = np.maximum(np.abs(b_).max(axis=1), 1e-300)
                rel = (np.abs(a - b_).max(axis=1) / den).max()
                worst = max(worst, rel)
        if gD.size:
            rel = np.abs(gD - oD).max() / max(np.abs(oD).max(), 1e-300)
            worst = max(worst, rel)
    if worst > tol:
        problems.append("max normwise relative difference %.3e > %.1e" % (worst, tol))
    return {"problems": problems, "max_rel": worst}


def overrides_from_near(near):
    """GPU near-threshold decisions -> oracle override list (blk, side, idx, keep)."""
    return [tuple(int(x) for x in row) for row in np.asarray(near)]


def assert_replay_bounded(of, overrides):
    """The decision replay (reading R15) may only touch near-threshold decisions: every
    override matched a decision of the oracle (which refuses, with an error, any override
    whose own margin exceeds 1e-6), and there are no more overrides than decisions the
    oracle itself finds within 1e-8 of tau."""
    n = len(overrides)
    assert of.n_override_applied == n, (of.n_override_applied, n)
    assert n <= of.n_near, (n, of.n_near)


def dense_LPU(f, n):
    """Dense L, P (= D^{-1} blocks), U of a factor (small n only; test helper)."""
    L = np.eye(n)
    U = np.eye(n)
    P = np.zeros((n, n))
    for K in range(f.nblk):
        s, e, rows, Lp, cols, Ut, D = f.block(K)
        if len(rows):
            L[np.asarray(rows)[:, None], np.arange(s, e)[None, :]] = Lp
        Pk = np.linalg.inv(D)
        P[s:e, s:e] = Pk
        if len(cols):
            U[np.arange(s, e)[:, None], np.asarray(cols)[None, :]] = D @ Ut
    return L, P, U


def compare_present_blocks(g, o, present_start, tol=1e-10):
    """compare_factors restricted to the final blocks of `o` that start at an index in
    `present_start` (the blocks a rank of the distributed factorization holds); each must
    exist in `g` with the same extent."""
    problems = []
    gstart = {int(s): K for K, s in enumerate(np.asarray(g.bstart)[:-1])}
    worst = 0.0
    checked = 0
    for K in range(o.nblk):
        s0 = int(o.bstart[K])
        if s0 not in present_start:
            continue
        if s0 not in gstart or int(g.bstart[gstart[s0] + 1]) != int(o.bstart[K + 1]):
            problems.append("block at %d: extent differs" % s0)
            continue
        s, e, gr, gL, gc, gU, gD = g.block(gstart[s0])
        _, _, orr, oL, oc, oU, oD = o.block(K)
        checked += 1
        if not np.array_equal(gr, orr) or not np.array_equal(gc, oc):
            problems.append("block at %d: pattern differs" % s0)
            continue
        for a, b_ in ((gL, oL), (gU.T, oU.T)):
            if a.size:
                den = np.maximum(np.abs(b_).max(axis=1), 1e-300)
                worst = max(worst, (np.abs(a - b_).max(axis=1) / den).max())
        if gD.size:
            worst = max(worst, np.abs(gD - oD).max() / max(np.abs(oD).max(), 1e-300))
    if worst > tol:
        problems.append("max normwise relative difference %.3e > %.1e" % (worst, tol))
    return {"problems": problems, "max_rel": worst, "checked": checked}


def oracle_replay(*args, overrides=None, **kw):
    """oracle.factor with the GPU's near-threshold decisions replayed (R15), bounded by
    assert_replay_bounded."""
    import oracle
    ov = list(overrides or [])
    of = oracle.factor(*args, overrides=ov, **kw)
    assert_replay_bounded(of, ov)
    return of
