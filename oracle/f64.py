"""float64 restatement of loss_and_grad (TEST INFRASTRUCTURE ONLY — a precision yardstick).

The same mathematics as oracle/ember_oracle.c orc_loss_and_grad (SPEC.md:139-165 with the sign
fix of SPEC.md:192; adjusted vectors as in ember_oracle.c:108-145), computed in float64 with numpy,
plus, for every output element, the sum of the absolute values of the terms that form it (M). An
fp32 computation of a sum of terms carries an error that scales with M, not with the value, so an
element whose value cancels (|value| << M) cannot be held to a relative bound by any fp32
implementation, the fp32 oracle included; tests report element-wise errors against this reference
relative to |value| and to M.

Only tests/ import this module.
"""
from __future__ import annotations

import numpy as np

KINDS = {"dot": 0, "distmult": 1, "complex": 2}


def _adjust(kind, x, r, side, absval=False):
    """side 0: adj_dst(s=x, r); side 1: adj_src(r, t=x). absval: the same formula on |.| (magnitudes)."""
    if absval:
        x, r = np.abs(x), (np.abs(r) if r is not None else None)
    if kind == 0:
        return x.copy()
    if kind == 1:
        return x * r
    h = x.shape[1] // 2
    a, b = x[:, :h], x[:, h:]
    c, e = r[:, :h], r[:, h:]
    if side == 0:  # (a + ib)(c + ie)
        re, im = a * c - b * e, a * e + b * c
        if absval:
            re, im = a * c + b * e, a * e + b * c
    else:  # [Re(r conj t) | -Im(r conj t)] with t = a + ib
        re, im = c * a + e * b, c * b - e * a
        if absval:
            re, im = c * a + e * b, c * b + e * a
    return np.concatenate([re, im], 1)


def _chain(kind, u, w, s, r, t, absval=False):
    """dL/ds, dL/dr, dL/dt from u = dL/d adj_dst, w = dL/d adj_src (ember_oracle.c chain rule)."""
    if absval:
        s, t = np.abs(s), np.abs(t)
        r = np.abs(r) if r is not None else None
    sg = -1.0 if not absval else 1.0
    if kind == 0:
        return u.copy(), None, w.copy()
    if kind == 1:
        return u * r, u * s + w * t, w * r
    h = s.shape[1] // 2
    a, b, c, e, x, y = s[:, :h], s[:, h:], r[:, :h], r[:, h:], t[:, :h], t[:, h:]
    u0, u1, w0, w1 = u[:, :h], u[:, h:], w[:, :h], w[:, h:]
    gS = np.concatenate([u0 * c + u1 * e, u1 * c + sg * u0 * e], 1)
    gR = np.concatenate([(u0 * a + u1 * b) + (w0 * x + w1 * y), (u1 * a + sg * u0 * b) + (w0 * y + sg * w1 * x)], 1)
    gT = np.concatenate([w0 * c + sg * w1 * e, w0 * e + w1 * c], 1)
    return gS, gR, gT


def _segment_sum(keys, rows):
    order = np.argsort(keys, kind="stable")
    k = keys[order]
    starts = np.flatnonzero(np.r_[True, k[1:] != k[:-1]])
    return k[starts], np.add.reduceat(rows[order], starts, axis=0)


def loss_and_grad(kind, edges, negs, node_theta, rel_theta, chunks=1):
    """edges (nb, 3) and negs (chunks*2*n_t,) index node_theta / rel_theta rows. Returns float64
    values and magnitudes: loss, fpos, lse (2, nb), node_ids / node_rows / node_mag, rel_ids /
    rel_rows / rel_mag (ids ascending, one summed row per id)."""
    kind = KINDS[kind] if isinstance(kind, str) else int(kind)
    e = np.asarray(edges, np.int64).reshape(-1, 3)
    nb = e.shape[0]
    th = np.asarray(node_theta, np.float64)
    rt = np.asarray(rel_theta, np.float64)
    negs = np.asarray(negs, np.int64)
    nt = negs.size // (2 * chunks)
    S_, R_, T_ = th[e[:, 0]], (rt[e[:, 1]] if kind else None), th[e[:, 2]]
    A = [_adjust(kind, S_, R_, 0), _adjust(kind, T_, R_, 1)]
    Am = [_adjust(kind, S_, R_, 0, True), _adjust(kind, T_, R_, 1, True)]
    other = [T_, S_]
    fpos = np.einsum("ij,ij->i", A[0], T_)
    chunk_rows = (nb + chunks - 1) // chunks
    dA = [np.zeros_like(A[0]), np.zeros_like(A[1])]
    dAm = [np.zeros_like(A[0]), np.zeros_like(A[1])]
    g0 = np.zeros((2, nb))
    lse = np.zeros((2, nb))
    dN = np.zeros((negs.size, th.shape[1]))
    dNm = np.zeros_like(dN)
    for q in range(chunks):
        e0, e1 = q * chunk_rows, min(nb, (q + 1) * chunk_rows)
        if e0 >= e1:
            continue
        for side in range(2):
            ids = negs[(2 * q + side) * nt:(2 * q + side + 1) * nt]
            N = th[ids]
            S = A[side][e0:e1] @ N.T
            f = fpos[e0:e1, None]
            mx = np.maximum(f, S.max(1, keepdims=True))
            Z = np.exp(f - mx) + np.exp(S - mx).sum(1, keepdims=True)
            L = (mx + np.log(Z))[:, 0]
            lse[side, e0:e1] = L
            P = np.exp(S - L[:, None]) / nb
            g0[side, e0:e1] = (np.exp(fpos[e0:e1] - L) - 1.0) / nb
            dA[side][e0:e1] = g0[side, e0:e1, None] * other[side][e0:e1] + P @ N
            dAm[side][e0:e1] = np.abs(g0[side, e0:e1, None]) * np.abs(other[side][e0:e1]) + P @ np.abs(N)
            sl = slice((2 * q + side) * nt, (2 * q + side + 1) * nt)
            dN[sl] = P.T @ A[side][e0:e1]
            dNm[sl] = P.T @ Am[side][e0:e1]
    loss = float(((lse[0] - fpos) + (lse[1] - fpos)).mean())
    gS, gR, gT = _chain(kind, dA[0], dA[1], S_, R_, T_)
    mS, mR, mT = _chain(kind, dAm[0], dAm[1], S_, R_, T_, absval=True)
    # positive-score terms: f = adj_dst . t and f = adj_src . s
    gT = gT + g0[0][:, None] * A[0]
    gS = gS + g0[1][:, None] * A[1]
    mT = mT + np.abs(g0[0])[:, None] * Am[0]
    mS = mS + np.abs(g0[1])[:, None] * Am[1]
    keys = np.concatenate([e[:, 0], e[:, 2], negs])
    node_ids, node_rows = _segment_sum(keys, np.concatenate([gS, gT, dN]))
    _, node_mag = _segment_sum(keys, np.concatenate([mS, mT, dNm]))
    out = {"loss": loss, "fpos": fpos, "fpos_mag": np.einsum("ij,ij->i", Am[0], np.abs(T_)), "lse": lse,
           "node_ids": node_ids.astype(np.uint32), "node_rows": node_rows, "node_mag": node_mag}
    if kind:
        rel_ids, rel_rows = _segment_sum(e[:, 1], gR)
        _, rel_mag = _segment_sum(e[:, 1], mR)
        out.update(rel_ids=rel_ids.astype(np.uint32), rel_rows=rel_rows, rel_mag=rel_mag)
    else:
        out.update(rel_ids=np.zeros(0, np.uint32), rel_rows=np.zeros((0, th.shape[1])),
                   rel_mag=np.zeros((0, th.shape[1])))
    return out


def elementwise(x, exact, mag, rtol=1e-4):
    """Element-wise error statistics of x against the float64 values `exact` with term magnitudes `mag`."""
    x = np.asarray(x, np.float64)
    err = np.abs(x - exact)
    ax = np.abs(exact)
    rel = err / np.maximum(ax, 1e-300)
    well = ax >= 0.1 * mag  # condition number |value| / M <= 10
    return {
        "n": int(x.size),
        "max_rel_well_conditioned": float(rel[well].max()) if well.any() else 0.0,
        "frac_well_conditioned": float(well.mean()),
        "frac_within_rtol": float((err <= rtol * ax).mean()),
        "max_err_over_mag": float((err / np.maximum(mag, 1e-300)).max()),
        "p99_rel": float(np.quantile(rel, 0.99)),
        "max_rel": float(rel.max()),
    }
