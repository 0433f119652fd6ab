"""Oracle: CPU fp64 Gaussian sums restricted to a ball, for full-size parity spot checks.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the exact sum of
_kernels_py.gauss_direct (/root/reference/pkg/src/fgt/_kernels_py.py:14-30; periodic
minimum image :33-46) over the sources near each target.  u(x) = sum_{|x-y| <= r} exp(-|x-y|^2/delta) q over ALL sources,
with r^2 = 40 delta (the dropped tail is < e^-40 ~ 4e-18 per unit charge, far below every
tolerance checked), found by binning the sources into cells of side >= r (numpy stable
argsort; the 3^d cells around each target).  Periodic mode uses the minimum image on the
unit cell (exact while delta << 1/4, i.e. the image regime of the configs).
"""

import numpy as np


def near_sum(src, q, tgt, delta, periodic=False, r2_factor=40.0):
    src = np.asarray(src, dtype=np.float64)
    tgt = np.asarray(tgt, dtype=np.float64)
    d = src.shape[1]
    r = float(np.sqrt(r2_factor * delta))
    lo = -0.5 if periodic else float(min(src.min(), tgt.min()))
    hi = 0.5 if periodic else float(max(src.max(), tgt.max()))
    span = hi - lo
    nc = max(1, int(np.floor(span / r)))
    nc = min(nc, int(round(1e8 ** (1.0 / d))))  # bounded cell table
    h = span / nc

    def cell(p):
        c = np.floor((p - lo) / h).astype(np.int64)
        return np.clip(c, 0, nc - 1)

    def keys(c):
        k = np.zeros(c.shape[0], dtype=np.int64)
        for a in range(d):
            k = k * nc + c[:, a]
        return k

    ct = cell(tgt)
    offs = np.stack(np.meshgrid(*([np.array([-1, 0, 1])] * d), indexing="ij"), -1).reshape(-1, d)
    # keep only the sources in cells next to some target (a table lookup over all sources)
    near = (ct[:, None, :] + offs[None]).reshape(-1, d)
    near = np.mod(near, nc) if periodic else np.clip(near, 0, nc - 1)
    want = np.zeros(nc ** d, dtype=bool)
    want[keys(near)] = True
    key = np.empty(src.shape[0], dtype=np.int64)
    for a in range(0, src.shape[0], 1 << 24):  # chunked: bounded temporaries at 10^8 points
        key[a:a + (1 << 24)] = keys(cell(src[a:a + (1 << 24)]))
    sel = np.nonzero(want[key])[0]
    key = key[sel]
    order = np.argsort(key, kind="stable")
    skey = key[order]
    ssrc = src[sel[order]]
    sq = np.asarray(q)[sel[order]]
    out = np.zeros(tgt.shape[0])
    inv = 1.0 / delta
    for i in range(tgt.shape[0]):
        c = ct[i] + offs
        if periodic:
            c = np.mod(c, nc)
        else:
            c = c[np.all((c >= 0) & (c < nc), axis=1)]
        c = np.unique(c, axis=0)
        kk = np.zeros(c.shape[0], dtype=np.int64)
        for k in range(d):
            kk = kk * nc + c[:, k]
        a = np.searchsorted(skey, kk, "left")
        b = np.searchsorted(skey, kk, "right")
        idx = np.concatenate([np.arange(s, e) for s, e in zip(a, b)]) if a.size else np.zeros(0, int)
        if idx.size == 0:
            continue
        diff = ssrc[idx] - tgt[i]
        if periodic:
            diff -= np.round(diff)
        r2 = np.einsum("ij,ij->i", diff, diff)
        m = r2 <= r * r
        out[i] = np.dot(np.exp(-r2[m] * inv), sq[idx[m]])
    return out
