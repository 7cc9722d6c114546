"""Pure-numpy model of the device integral pipeline's carry algebra (test helper).

It restates, tile by tile, what csrc/integral.cu computes -- the per-tile aggregates
(reduce), the float64 carry recurrences over bands (scan) and the per-pixel assembly
of rect_tl / wedge_up plus the six derived tables (write) -- so the decomposition can
be checked against the oracle on the CPU, independently of the CUDA code.
"""

from __future__ import annotations

import numpy as np


def _chains(V):
    """In-tile up-left / up-right chains of the column prefix V (clipped at the tile)."""
    TH, TW = V.shape
    UL = np.zeros_like(V)
    UR = np.zeros_like(V)
    for r in range(TH):
        prevL = np.zeros(TW) if r == 0 else np.concatenate([[0.0], UL[r - 1, :-1]])
        prevR = np.zeros(TW) if r == 0 else np.concatenate([UR[r - 1, 1:], [0.0]])
        UL[r] = V[r] + prevL
        UR[r] = V[r] + prevR
    return UL, UR


def geometry(s: int):
    TH = s if s < 16 else (16 if s <= 2048 else 32)
    TW = 256 if s >= 8192 else (s if s < 128 else 128)
    return TH, TW


def model_tables(d: np.ndarray, TH: int | None = None, TW: int | None = None):
    d = np.asarray(d, dtype=np.float64)
    s = d.shape[0]
    gTH, gTW = geometry(s)
    TH = TH or gTH
    TW = TW or gTW
    B, NX = s // TH, s // TW
    colsum = np.zeros((B, s))
    rowsum = np.zeros((s, NX))
    ulbot = np.zeros((B, s))
    urbot = np.zeros((B, s))
    ule = np.zeros((B, NX, TH))
    ure = np.zeros((B, NX, TH))
    # ---- reduce
    for b in range(B):
        a = b * TH
        for x in range(NX):
            i0 = x * TW
            tile = d[a:a + TH, i0:i0 + TW]
            V = np.cumsum(tile, axis=0)
            UL, UR = _chains(V)
            colsum[b, i0:i0 + TW] = V[-1]
            rowsum[a:a + TH, x] = tile.sum(axis=1)
            ulbot[b, i0:i0 + TW] = UL[-1]
            urbot[b, i0:i0 + TW] = UR[-1]
            ule[b, x] = UL[:, -1]
            ure[b, x] = UR[:, 0]
    # ---- scan
    ulb2 = ulbot.copy()
    urb2 = urbot.copy()
    for b in range(B):
        for c in range(s):
            x, u = divmod(c, TW)
            rr = TH - 2 - u
            if x > 0 and rr >= 0:
                ulb2[b, c] += ule[b, x - 1, rr]
            rq = TH - 1 - (TW - u)
            if x < NX - 1 and rq >= 0:
                urb2[b, c] += ure[b, x + 1, rq]
    # band-local row prefix of the column sums, as the device forms it: tile-level
    # exclusive prefix of the tile totals + the in-tile prefix written by the reduce
    inpre = np.zeros((B, s))
    tiletot = np.zeros((B, NX))
    for b in range(B):
        for x in range(NX):
            seg = colsum[b, x * TW:(x + 1) * TW]
            inpre[b, x * TW:(x + 1) * TW] = np.cumsum(seg)
            tiletot[b, x] = seg.sum()
    tilepre = np.concatenate([np.zeros((B, 1)), np.cumsum(tiletot, axis=1)[:, :-1]], axis=1)
    batl = tilepre[:, np.arange(s) // TW] + inpre
    bandpre = np.concatenate([[0.0], np.cumsum(tiletot.sum(axis=1))])  # TLcar_b[s-1]
    tlcar = np.vstack([np.zeros((1, s)), np.cumsum(batl, axis=0)])

    # X1 = ULcar - TLcar and X2 = URcar + TLcar[c-1] as sheared scans of band-local terms:
    #   X1_{b+1}[c] = X1_b[c-TH] + ULbot2_b[c] - batl_b[c]
    #   X2_{b+1}[c] = X2_b[c+TH] + URbot2_b[c] + batl_b[c-1],  X2_b[c >= s] = TLcar_b[s-1]
    X1 = np.zeros((B + 1, s))
    X2 = np.zeros((B + 1, s))
    for b in range(B):
        for c in range(s):
            X1[b + 1, c] = (X1[b, c - TH] if c - TH >= 0 else 0.0) + ulb2[b, c] - batl[b, c]
            X2[b + 1, c] = ((X2[b, c + TH] if c + TH < s else bandpre[b]) + urb2[b, c]
                            + (batl[b, c - 1] if c >= 1 else 0.0))
    x1 = X1[:B]
    x2 = np.zeros((B, s + TH))
    for b in range(B):
        x2[b, :s] = X2[b]
        x2[b, s:] = bandpre[b]
    hc = np.concatenate([np.zeros((s, 1)), np.cumsum(rowsum, axis=1)[:, :-1]], axis=1)
    rtot = rowsum.sum(axis=1)
    rpre = np.array([bandpre[j // TH] + rtot[(j // TH) * TH:j + 1].sum() for j in range(s)])
    cpre = tlcar[B]
    C = bandpre[B]
    # diagonal / anti-diagonal marginals from the chains (no per-tile partial sums):
    #   Dsuf[delta>=0] = UL[s-1-delta][s-1],  Dsuf[delta<0] = UL[s-1][s-1+delta] + C - Cpre[s-1+delta]
    #   Apre[sigma<s]  = UR[sigma][0],        Apre[sigma>=s] = UR[s-1][sigma-s+1] + Cpre[sigma-s]
    dsuf = np.zeros(2 * s - 1)
    apre = np.zeros(2 * s - 1)
    for q in range(2 * s - 1):
        delta = q - (s - 1)
        if delta >= 0:
            j = s - 1 - delta
            b, r = divmod(j, TH)
            c2 = s - 2 - r
            dsuf[q] = ule[b, NX - 1, r] + bandpre[b] + (x1[b, c2] if c2 >= 0 else 0.0)
        else:
            dsuf[q] = X1[B, s - 1 + delta] + C           # ULrow + C - Cpre
        sigma = q
        if sigma < s:
            b, r = divmod(sigma, TH)
            apre[q] = ure[b, 0, r] + x2[b, r + 1]
        else:
            apre[q] = X2[B, sigma - (s - 1)]             # URrow + Cpre
    # ---- write
    out = np.zeros((8, s, s))
    for b in range(B):
        a = b * TH
        for x in range(NX):
            i0 = x * TW
            tile = d[a:a + TH, i0:i0 + TW]
            V = np.cumsum(tile, axis=0)
            UL, UR = _chains(V)
            for r in range(TH):
                for u in range(TW):
                    re = r - u - 1
                    if re >= 0 and x > 0:
                        UL[r, u] += ule[b, x - 1, re]
                    rq = r - (TW - u)
                    if rq >= 0 and x < NX - 1:
                        UR[r, u] += ure[b, x + 1, rq]
            T = UL + UR - V
            local = np.cumsum(V, axis=1)
            vh = np.cumsum(hc[a:a + TH, x])
            for r in range(TH):
                j = a + r
                h = r + 1
                for u in range(TW):
                    i = i0 + u
                    tl = tlcar[b, i] + vh[r] + local[r, u]
                    up = T[r, u] + (x1[b, i - h] if i - h >= 0 else 0.0) + x2[b, i + h]
                    Rp, Cp, Ap, Ds = rpre[j], cpre[i], apre[i + j], dsuf[i - j + s - 1]
                    out[:, j, i] = (tl, Cp - tl, C - Rp - Cp + tl, Rp - tl, up, Ap - up, C - Ap - Ds + up, Ds - up)
    return out, C
