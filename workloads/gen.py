"""Synthetic inputs for the BASELINE.json configs (SURVEY.md 8(d) generator rules).

* SplitMix64 counter generator, vectorised in numpy: doubles from the top 53
  bits, no libstdc++ distributions -- the same arrays feed the oracle and the
  GPU, so nothing has to be regenerated consistently across languages.
* CSR rows are built directly, sorted ascending, no duplicates (the format
  from_triplets produces, split.cpp:15-33).
* Seeds: 0x200907495 ^ cfg_id.

The paper's SuiteSparse matrices are not available offline; these seeded
stencils / random matrices stand in with the shapes BASELINE.json names.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 0x200907495
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """count outputs of SplitMix64 starting at stream position offset."""
    with np.errstate(over="ignore"):
        idx = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, count: int, lo: float = -1.0, hi: float = 1.0, offset: int = 0) -> np.ndarray:
    u = (splitmix64(seed, count, offset) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return lo + (hi - lo) * u


def uniform_int(seed: int, count: int, lo: int, hi: int, offset: int = 0) -> np.ndarray:
    """integers uniform in [lo, hi] (inclusive); hi - lo < 2^63."""
    span = np.uint64(hi - lo + 1)
    r = splitmix64(seed, count, offset) % span
    return (r.astype(np.int64) + np.int64(lo)).astype(np.int64)


def normal(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """Box-Muller normals."""
    m = (count + 1) // 2
    u1 = uniform(seed, m, 0.0, 1.0, offset)
    u2 = uniform(seed, m, 0.0, 1.0, offset + m)
    u1 = np.where(u1 <= 0.0, 2.0 ** -53, u1)
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.concatenate([r * np.cos(2 * np.pi * u2), r * np.sin(2 * np.pi * u2)])
    return z[:count]


# ---------------------------------------------------------------- stencils
def _stencil_csr(dims, offsets, coef_fn):
    """CSR of a structured-grid stencil in natural order (x fastest).

    offsets: list of (di, dj, dk) sorted so that the flat column offsets are
    ascending; coef_fn(offset_index, valid_mask, rows) -> values for those rows.
    Out-of-grid neighbours are dropped (Dirichlet).
    """
    gx, gy, gz = dims
    n = gx * gy * gz
    r = np.arange(n, dtype=np.int64)
    i = r % gx
    j = (r // gx) % gy
    k = r // (gx * gy)
    flat = [dk * gx * gy + dj * gx + di for (di, dj, dk) in offsets]
    order = np.argsort(flat, kind="stable")
    masks, cols, vals = [], [], []
    for o in order:
        di, dj, dk = offsets[o]
        ok = ((i + di >= 0) & (i + di < gx) & (j + dj >= 0) & (j + dj < gy) & (k + dk >= 0) & (k + dk < gz))
        masks.append(ok)
        cols.append((r + flat[o]).astype(np.int64))
        vals.append(coef_fn(o, r))
    mask = np.stack(masks, axis=1)
    counts = mask.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col = np.stack(cols, axis=1)[mask].astype(np.int32)
    val = np.stack(vals, axis=1)[mask].astype(np.float64)
    return row_ptr.astype(np.int32), col, val


def upwind_2d(g: int, beta=(10.0, 10.0)):
    """Config 1: -Lap u + beta.grad u, 5-point first-order upwind, h = 1/(g+1)."""
    h = 1.0 / (g + 1)
    d = 4.0 / h ** 2 + (beta[0] + beta[1]) / h
    offs = [(0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0)]
    upw = {0: -1.0 / h ** 2 - beta[1] / h, 1: -1.0 / h ** 2 - beta[0] / h, 2: d,
           3: -1.0 / h ** 2, 4: -1.0 / h ** 2}
    return _stencil_csr((g, g, 1), offs, lambda o, r: np.full(r.shape, upw[o]))


def upwind_3d(g: int, beta: float = 20.0):
    """Configs 2 / 5: 7-point upwind convection-diffusion, h = 1/(g+1)."""
    h = 1.0 / (g + 1)
    d = 6.0 / h ** 2 + 3 * beta / h
    offs = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    coef = {0: -1.0 / h ** 2 - beta / h, 1: -1.0 / h ** 2 - beta / h, 2: -1.0 / h ** 2 - beta / h,
            3: d, 4: -1.0 / h ** 2, 5: -1.0 / h ** 2, 6: -1.0 / h ** 2}
    return _stencil_csr((g, g, g), offs, lambda o, r: np.full(r.shape, coef[o]))


def stencil27(g: int, seed: int):
    """Config 4: 27-point, off-diagonals -u*(1+0.1*sigma(d)), u~U[0,1), a_rr = 1.05*sum|a_rd|."""
    offs = [(di, dj, dk) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]
    n = g ** 3

    def coef(o, r):
        di, dj, dk = offs[o]
        if (di, dj, dk) == (0, 0, 0):
            return np.zeros(r.shape)
        s = di + dj + dk
        sig = 1.0 if s < 0 else (-1.0 if s > 0 else 0.0)
        u = uniform(seed, n, 0.0, 1.0, offset=o * n)
        return -u * (1.0 + 0.1 * sig)

    rp, ci, v = _stencil_csr((g, g, g), offs, coef)
    rows = np.repeat(np.arange(n), np.diff(rp))
    diag = ci == rows
    rs = np.bincount(rows, weights=np.abs(v), minlength=n)
    v[diag] = 1.05 * rs
    return rp, ci, v


def random_band(n: int, seed: int, band: int = 2, extra: int = 10):
    """Config 3: band i-2..i+2 plus `extra` distinct random columns outside the band."""
    cols = []
    base = np.arange(n, dtype=np.int64)[:, None] + np.arange(-band, band + 1)[None, :]
    rnd = uniform_int(seed, n * extra * 2, 0, n - 1).reshape(n, extra * 2)
    rows = []
    for i in range(n):  # only used at small sizes in tests; bench builds it vectorised later
        c = set(int(x) for x in base[i] if 0 <= x < n)
        band_set = set(c)
        for x in rnd[i]:
            if len(c) >= len(band_set) + extra:
                break
            if int(x) not in c:
                c.add(int(x))
        rows.append(sorted(c))
    rp = np.zeros(n + 1, dtype=np.int32)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.concatenate([np.array(r, dtype=np.int32) for r in rows])
    offd = normal(seed ^ 0xABCDEF, len(ci))
    rr = np.repeat(np.arange(n), np.diff(rp))
    diag = ci == rr
    offd[diag] = 0.0
    rs = np.bincount(rr, weights=np.abs(offd), minlength=n)
    offd[diag] = 1.2 * rs
    return rp, ci, offd


def spmv_np(rp, ci, v, x):
    """y = A x in numpy (generator helper: builds b = A x*)."""
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    return np.bincount(rows, weights=v * x[ci], minlength=len(rp) - 1)


# ---------------------------------------------------------------- small test matrices
def laplacian2d(g: int):
    """5-point Laplacian (4 on the diagonal, -1 off), natural order."""
    offs = [(0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0)]
    return _stencil_csr((g, g, 1), offs, lambda o, r: np.full(r.shape, 4.0 if o == 2 else -1.0))


def random_dominant(n: int, density: float, dominance: float, seed: int):
    """Random sparse matrix, diagonal = dominance * (row abs sum + 0.25)."""
    coin = uniform(seed, n * n, 0.0, 1.0).reshape(n, n)
    val = uniform(seed ^ 0x55, n * n, -1.0, 1.0).reshape(n, n)
    mask = coin < density
    np.fill_diagonal(mask, False)
    dense = np.where(mask, val, 0.0)
    rs = np.abs(dense).sum(axis=1)
    dense[np.arange(n), np.arange(n)] = dominance * (rs + 0.25)
    mask[np.arange(n), np.arange(n)] = True
    rp = np.zeros(n + 1, dtype=np.int32)
    rp[1:] = np.cumsum(mask.sum(axis=1))
    rr, cc = np.nonzero(mask)
    return rp, cc.astype(np.int32), dense[rr, cc].astype(np.float64)


def upwind_3d_lean(g: int, beta: float = 20.0):
    """upwind_3d() for large grids (config 5: 400^3) without n x 7 temporaries.

    Same matrix, row for row, as upwind_3d(); rows are filled offset by
    offset in ascending column order."""
    h = 1.0 / (g + 1)
    n = g * g * g
    d = 6.0 / h ** 2 + 3 * beta / h
    lo, hi = -1.0 / h ** 2 - beta / h, -1.0 / h ** 2
    r = np.arange(n, dtype=np.int64)
    i = (r % g).astype(np.int32)
    j = ((r // g) % g).astype(np.int32)
    k = (r // (g * g)).astype(np.int32)
    del r
    offs = [(k > 0, -g * g, lo), (j > 0, -g, lo), (i > 0, -1, lo), (None, 0, d),
            (i < g - 1, 1, hi), (j < g - 1, g, hi), (k < g - 1, g * g, hi)]
    counts = np.full(n, 1, dtype=np.int32)
    for m, _, _ in offs:
        if m is not None:
            counts += m
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    del counts
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    cur = row_ptr[:-1].copy()
    for m, off, c in offs:
        idx = np.arange(n, dtype=np.int64) if m is None else np.nonzero(m)[0]
        pos = cur[idx]
        col[pos] = (idx + off).astype(np.int32)
        val[pos] = c
        cur[idx] += 1
        del idx, pos
    return row_ptr.astype(np.int32), col, val


def device_uniform_int40(n: int, seed: int, offset: int, device="cuda"):
    """Seeded SplitMix64 on the device (torch int64, wrapping), mapped to
    integers uniform in [-2^40, 2^40): config 5's vector distribution
    (bench_kernels.cpp:14-21 uses +-2^40)."""
    import torch
    to_i64 = lambda u: int(np.uint64(u).view(np.int64))
    gold, m1, m2 = to_i64(0x9E3779B97F4A7C15), to_i64(0xBF58476D1CE4E5B9), to_i64(0x94D049BB133111EB)
    z = torch.arange(offset + 1, offset + n + 1, dtype=torch.int64, device=device)
    z = z * gold + to_i64(seed & 0xFFFFFFFFFFFFFFFF)
    z = (z ^ ((z >> 30) & ((1 << 34) - 1))) * m1
    z = (z ^ ((z >> 27) & ((1 << 37) - 1))) * m2
    z = z ^ ((z >> 31) & ((1 << 33) - 1))
    return ((z >> 23) & ((1 << 41) - 1)) - (1 << 40)


def upwind_3d_slab(g: int, beta: float, z0: int, z1: int):
    """Planes [z0, z1) of upwind_3d(g) as an extended-square local CSR for
    row-block partitioning: the local index space is the
    halo range of planes [max(0, z0-1), min(g, z1+1)); rows of the halo
    planes are empty, rows of the own planes are upwind_3d's rows with
    columns shifted into the local space.  Returns (row_ptr, col, val,
    h0, own0, own1) with h0 = first global row of the local space and
    [own0, own1) the own rows in local indices."""
    zh0, zh1 = max(0, z0 - 1), min(g, z1 + 1)
    p = g * g
    h0 = zh0 * p
    nl = (zh1 - zh0) * p
    own0, own1 = (z0 - zh0) * p, (z1 - zh0) * p
    h = 1.0 / (g + 1)
    d = 6.0 / h ** 2 + 3 * beta / h
    lo, hi = -1.0 / h ** 2 - beta / h, -1.0 / h ** 2
    r = np.arange(z0 * p, z1 * p, dtype=np.int64)  # own global rows
    i = (r % g).astype(np.int32)
    j = ((r // g) % g).astype(np.int32)
    k = (r // p).astype(np.int32)
    offs = [(k > 0, -p, lo), (j > 0, -g, lo), (i > 0, -1, lo), (None, 0, d),
            (i < g - 1, 1, hi), (j < g - 1, g, hi), (k < g - 1, p, hi)]
    no = len(r)
    counts = np.full(no, 1, dtype=np.int32)
    for m, _, _ in offs:
        if m is not None:
            counts += m
    row_ptr = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[own0 + 1:own1 + 1])
    row_ptr[own1 + 1:] = row_ptr[own1]
    nnz = int(row_ptr[own1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    cur = row_ptr[own0:own1].copy()
    for m, off, c in offs:
        idx = np.arange(no, dtype=np.int64) if m is None else np.nonzero(m)[0]
        pos = cur[idx]
        col[pos] = (r[idx] + off - h0).astype(np.int32)
        val[pos] = c
        cur[idx] += 1
    return row_ptr.astype(np.int32), col, val, h0, own0, own1


def stencil27_lean(g: int, seed: int):
    """stencil27() for large grids (config 4: 256^3) without n x 27
    temporaries: the same arrays, entry for entry (rows filled offset by
    offset in ascending column order; the diagonal's row sum accumulated in
    the same left-to-right order as stencil27's bincount)."""
    n = g ** 3
    p = g * g
    r = np.arange(n, dtype=np.int64)
    i = (r % g).astype(np.int16)
    j = ((r // g) % g).astype(np.int16)
    k = (r // p).astype(np.int16)
    del r
    offs = [(di, dj, dk) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]

    def ok(di, dj, dk):
        m = np.ones(n, dtype=bool)
        for c, d in ((i, di), (j, dj), (k, dk)):
            if d < 0:
                m &= c > 0
            elif d > 0:
                m &= c < g - 1
        return m

    counts = np.zeros(n, dtype=np.int32)
    for (di, dj, dk) in offs:
        counts += ok(di, dj, dk)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    del counts
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    cur = row_ptr[:-1].copy()
    rs = np.zeros(n)
    dpos = None
    for o, (di, dj, dk) in enumerate(offs):
        m = ok(di, dj, dk)
        idx = np.nonzero(m)[0]
        pos = cur[idx]
        col[pos] = (idx + (dk * p + dj * g + di)).astype(np.int32)
        if (di, dj, dk) == (0, 0, 0):
            val[pos] = 0.0
            dpos = pos
        else:
            s = di + dj + dk
            sig = 1.0 if s < 0 else (-1.0 if s > 0 else 0.0)
            u = uniform(seed, n, 0.0, 1.0, offset=o * n)
            v = -u[idx] * (1.0 + 0.1 * sig)
            val[pos] = v
            a = np.zeros(n)
            a[idx] = np.abs(v)
            rs += a
            del u, v, a
        cur[idx] += 1
        del m, idx, pos
    val[dpos] = 1.05 * rs
    return row_ptr.astype(np.int32), col, val


def random_band_fast(n: int, seed: int, band: int = 2, extra: int = 10):
    """random_band() vectorised (config 3 at n = 1M): the same matrix.  Per
    row the candidates rnd[i, :] are taken in order, skipping band members
    and repeats, until `extra` were added."""
    cand = uniform_int(seed, n * extra * 2, 0, n - 1).reshape(n, extra * 2)
    rows = np.arange(n, dtype=np.int64)[:, None]
    new = np.abs(cand - rows) > band
    for t in range(1, cand.shape[1]):
        new[:, t] &= ~np.any(cand[:, :t] == cand[:, t:t + 1], axis=1)
    new &= np.cumsum(new, axis=1) <= extra
    bandc = rows + np.arange(-band, band + 1)[None, :]
    inb = (bandc >= 0) & (bandc < n)
    big = np.iinfo(np.int64).max
    allc = np.concatenate([np.where(inb, bandc, big), np.where(new, cand, big)], axis=1)
    allc.sort(axis=1)
    keep = allc != big
    counts = keep.sum(axis=1)
    rp = np.zeros(n + 1, dtype=np.int32)
    rp[1:] = np.cumsum(counts)
    ci = allc[keep].astype(np.int32)
    del allc, keep, cand, new
    offd = normal(seed ^ 0xABCDEF, len(ci))
    rr = np.repeat(np.arange(n), np.diff(rp))
    diag = ci == rr
    offd[diag] = 0.0
    rs = np.bincount(rr, weights=np.abs(offd), minlength=n)
    offd[diag] = 1.2 * rs
    return rp, ci, offd


# ---------------------------------------------------------------- plane-range generators
# Rows of whole z-planes [z0, z1) of the global matrices, with GLOBAL column
# indices, entry for entry equal to the rows of the whole-matrix generators: a
# z-slab rank builds only its own rows (dist.setup_slab_local).
def upwind_3d_rows(g: int, beta: float, z0: int, z1: int):
    """rows of planes [z0, z1) of upwind_3d(g, beta): (row_ptr, col (global), val)"""
    rp, ci, v, h0, own0, own1 = upwind_3d_slab(g, beta, z0, z1)
    a = int(rp[own0])
    return (rp[own0:own1 + 1] - a).astype(np.int32), (ci.astype(np.int64) + h0).astype(np.int32), v


def stencil27_rows(g: int, seed: int, z0: int, z1: int):
    """rows of planes [z0, z1) of stencil27(g, seed): (row_ptr, col (global), val).
    The per-offset uniform streams are indexed by global row (SplitMix64 is
    counter based), the diagonal's row sum accumulates in offset order as in
    stencil27_lean."""
    n, p = g ** 3, g * g
    r = np.arange(z0 * p, z1 * p, dtype=np.int64)
    no = len(r)
    i, j, k = r % g, (r // g) % g, r // p
    offs = [(di, dj, dk) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]

    def ok(di, dj, dk):
        m = np.ones(no, dtype=bool)
        for c, d in ((i, di), (j, dj), (k, dk)):
            if d < 0:
                m &= c > 0
            elif d > 0:
                m &= c < g - 1
        return m

    counts = np.zeros(no, dtype=np.int64)
    for o in offs:
        counts += ok(*o)
    row_ptr = np.zeros(no + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    cur = row_ptr[:-1].copy()
    rs = np.zeros(no)
    dpos = None
    for o, (di, dj, dk) in enumerate(offs):
        idx = np.nonzero(ok(di, dj, dk))[0]
        pos = cur[idx]
        col[pos] = (r[idx] + (dk * p + dj * g + di)).astype(np.int32)
        if (di, dj, dk) == (0, 0, 0):
            val[pos] = 0.0
            dpos = pos
        else:
            s = di + dj + dk
            sig = 1.0 if s < 0 else (-1.0 if s > 0 else 0.0)
            u = uniform(seed, no, 0.0, 1.0, offset=o * n + z0 * p)
            v = -u[idx] * (1.0 + 0.1 * sig)
            val[pos] = v
            a = np.zeros(no)
            a[idx] = np.abs(v)
            rs += a
        cur[idx] += 1
    val[dpos] = 1.05 * rs
    return row_ptr.astype(np.int32), col, val
