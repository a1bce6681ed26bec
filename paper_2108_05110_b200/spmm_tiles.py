"""Host-side tiling of the saddle SpMM for the tile-staged kernel (csrc/ens_spmm_tiles.cu).

Built once per mesh and member count.  Rows (velocity nodes, then pressure
rows, in the engine's internal order) are cut into tiles of consecutive rows
whose stage -- every neighbour segment the tile's rows touch, for both
sub-step systems, plus the tile's slices of the CSR streams -- fits one
shared-memory pipeline stage.  Each tile is described by

* a 16 x int32 descriptor: kind (0 velocity rows, 1 pressure rows), row range,
  its copy records, stage bytes, the per-system segment size, and for every
  staged stream the shared-memory "origin" offset o such that global element k
  of that stream sits at stage byte o + k * itemsize;
* bulk-copy records (int64 source byte offset from the stream's base, int32
  stage byte offset, int32 bytes | kind << 24); consecutive neighbour ids are
  merged into one copy;
* tile-local column slots for A_s (lcol_a), B^T (lcol_bt) and B (lcol_b).

Record kinds: 0 the iterate block X (2 x n_total x J), 1 A_s values (2 x nnz),
2 s_rowptr, 3 lcol_a, 4 bt_rowptr, 5 lcol_bt, 6 bt_val, 7 b_rowptr, 8 lcol_b,
9 b_val.
"""

from __future__ import annotations

import numpy as np

REC_DTYPE = np.dtype([("src", "<i8"), ("dst", "<i4"), ("bk", "<i4")])


def _a16(x):
    return (np.asarray(x, dtype=np.int64) + 15) & ~np.int64(15)


def _f16(x):
    return np.asarray(x, dtype=np.int64) & ~np.int64(15)


def _stream_bytes(first, last, item):
    """Aligned byte span of elements [first, last) (16-byte aligned start and end)."""
    return _a16(np.asarray(last, np.int64) * item) - _f16(np.asarray(first, np.int64) * item)


def _unique_per_tile(tile_of, cols, ncol):
    key = tile_of.astype(np.int64) * ncol + cols.astype(np.int64)
    return np.unique(key)


def _tile_sizes(bnd, rowptrs, colss, ncols, widths, items, J):
    """Stage bytes of every tile for boundaries ``bnd`` (both systems, streams included)."""
    ntile = len(bnd) - 1
    seg = np.zeros(ntile, np.int64)
    for rp, cols, ncol, w in zip(rowptrs, colss, ncols, widths):
        nrows = len(rp) - 1
        row_tile = np.searchsorted(bnd, np.arange(nrows), side="right") - 1
        tile_of = np.repeat(row_tile, np.diff(rp))
        u = _unique_per_tile(tile_of, cols, ncol)
        cnt = np.bincount(u // ncol, minlength=ntile)
        seg += cnt * w * 8
    total = 2 * seg
    r0, r1 = bnd[:-1], bnd[1:]
    for rp, its in zip(rowptrs, items):
        total = total + _stream_bytes(r0, r1 + 1, 4)          # row-pointer slice
        k0, k1 = rp[r0].astype(np.int64), rp[r1].astype(np.int64)
        for it, off in its:
            total = total + _stream_bytes(k0 + off, k1 + off, it)
    return total


def _cut(nrows, rows0, cap, rowptrs, colss, ncols, widths, items, J):
    bnd = np.unique(np.concatenate([np.arange(0, nrows, rows0), [nrows]])).astype(np.int64)
    for _ in range(64):
        sz = _tile_sizes(bnd, rowptrs, colss, ncols, widths, items, J)
        over = (sz > cap) & (np.diff(bnd) > 1)
        if not over.any():
            if (sz > cap).any():
                raise ValueError("a single SpMM row does not fit one tile stage")
            return bnd, sz
        mids = (bnd[:-1][over] + bnd[1:][over]) // 2
        bnd = np.unique(np.concatenate([bnd, mids]))
    raise RuntimeError("SpMM tiling did not converge")


def _runs(u, ncol, off):
    """Runs of consecutive ids in the per-tile sorted unique key list -> (tile, first id, slot, length)."""
    tile = u // ncol
    ids = u % ncol
    brk = np.ones(len(u), bool)
    brk[1:] = (tile[1:] != tile[:-1]) | (ids[1:] != ids[:-1] + 1)
    starts = np.flatnonzero(brk)
    lens = np.diff(np.concatenate([starts, [len(u)]]))
    return tile[starts], ids[starts], starts - off[tile[starts]], lens


def build_tiles(hm, J: int, cap: int = 64 * 1024, rows0: int = 64):
    """Tile the saddle SpMM of HostMesh ``hm`` for J member columns (J even, <= 64)."""
    if J % 2 or J > 64:
        raise ValueError("tile-staged SpMM needs an even J <= 64")
    ns, npres = hm.ns, hm.npres
    N = hm.ntot
    nvel = hm.nvel
    nnz = hm.nnz_s
    W2 = 2 * J
    # velocity tiles: neighbour nodes (2J doubles) + pressure rows (J doubles)
    vb, vsz = _cut(ns, rows0, cap, [hm.s_rowptr, hm.bt_rowptr], [hm.s_col, hm.bt_col], [ns, npres], [W2, J],
                   [((4, 0), (8, 0), (8, nnz)), ((4, 0), (16, 0))], J)
    pb, psz = _cut(npres, rows0, cap, [hm.b_rowptr], [hm.b_col], [ns], [W2], [((4, 0), (16, 0))], J)
    nvt, npt = len(vb) - 1, len(pb) - 1
    ntile = nvt + npt
    desc = np.zeros((ntile, 16), np.int32)
    recs = []   # (tile, order, src, dst, bytes, kind)

    def add(tile, order, src, dst, nbytes, kind):
        n = len(np.atleast_1d(tile))
        recs.append(np.rec.fromarrays([np.broadcast_to(np.asarray(tile, np.int64), (n,)),
                                       np.broadcast_to(np.asarray(order, np.int64), (n,)),
                                       np.broadcast_to(np.asarray(src, np.int64), (n,)),
                                       np.broadcast_to(np.asarray(dst, np.int64), (n,)),
                                       np.broadcast_to(np.asarray(nbytes, np.int64), (n,)),
                                       np.broadcast_to(np.asarray(kind, np.int64), (n,))],
                                      names="tile,order,src,dst,nb,kind"))

    def stream(tiles, order, kind, first, last, item, cursor, extra=0):
        """Stage a stream slice at ``cursor``; returns (origin offsets, new cursor)."""
        sb = _f16(first * item)
        nb = _stream_bytes(first, last, item)
        add(tiles, order, sb, cursor, nb, kind)
        return (cursor - sb + extra).astype(np.int64), cursor + nb

    # ---- velocity tiles
    r0, r1 = vb[:-1], vb[1:]
    vt = np.arange(nvt)
    row_tile = np.searchsorted(vb, np.arange(ns), side="right") - 1
    tile_a = np.repeat(row_tile, np.diff(hm.s_rowptr))
    ua = _unique_per_tile(tile_a, hm.s_col, ns)
    offa = np.searchsorted(ua // ns, np.arange(nvt + 1))
    lcol_a = (np.searchsorted(ua, tile_a * ns + hm.s_col) - offa[tile_a]).astype(np.int32)
    nv = np.diff(offa)
    tile_bt = np.repeat(row_tile, np.diff(hm.bt_rowptr))
    ubt = _unique_per_tile(tile_bt, hm.bt_col, npres)
    offbt = np.searchsorted(ubt // npres, np.arange(nvt + 1))
    lcol_bt = (np.searchsorted(ubt, tile_bt * npres + hm.bt_col) - offbt[tile_bt]).astype(np.int32)
    npv = np.diff(offbt)
    segsys_v = (nv * W2 + npv * J) * 8
    o_pres_v = nv * W2 * 8
    t_, id_, slot, ln = _runs(ua, ns, offa)
    for m in range(2):
        add(t_, 0, (m * N * J + id_ * W2) * 8, m * segsys_v[t_] + slot * W2 * 8, ln * W2 * 8, 0)
    if len(ubt):
        t_, id_, slot, ln = _runs(ubt, npres, offbt)
        for m in range(2):
            add(t_, 1, (m * N * J + (nvel + id_) * J) * 8, m * segsys_v[t_] + o_pres_v[t_] + slot * J * 8,
                ln * J * 8, 0)
    cur = 2 * segsys_v
    k0, k1 = hm.s_rowptr[r0].astype(np.int64), hm.s_rowptr[r1].astype(np.int64)
    q0, q1 = hm.bt_rowptr[r0].astype(np.int64), hm.bt_rowptr[r1].astype(np.int64)
    o_rp, cur = stream(vt, 2, 2, r0, r1 + 1, 4, cur)
    o_col, cur = stream(vt, 3, 3, k0, k1, 4, cur)
    o_a0, cur = stream(vt, 4, 1, k0, k1, 8, cur)
    o_a1, cur = stream(vt, 5, 1, k0 + nnz, k1 + nnz, 8, cur, extra=nnz * 8)
    o_btp, cur = stream(vt, 6, 4, r0, r1 + 1, 4, cur)
    o_btl, cur = stream(vt, 7, 5, q0, q1, 4, cur)
    o_btv, cur = stream(vt, 8, 6, q0, q1, 16, cur)
    assert np.array_equal(cur, vsz), "velocity tile sizes disagree"
    desc[:nvt, 0] = 0
    desc[:nvt, 1], desc[:nvt, 2] = r0, r1
    desc[:nvt, 5] = cur
    desc[:nvt, 6], desc[:nvt, 7] = segsys_v, o_pres_v
    for j, o in zip(range(8, 15), (o_rp, o_col, o_a0, o_a1, o_btp, o_btl, o_btv)):
        desc[:nvt, j] = o
    # ---- pressure tiles
    p0, p1 = pb[:-1], pb[1:]
    pt = nvt + np.arange(npt)
    prow_tile = np.searchsorted(pb, np.arange(npres), side="right") - 1
    tile_b = np.repeat(prow_tile, np.diff(hm.b_rowptr))
    ub = _unique_per_tile(tile_b, hm.b_col, ns)
    offb = np.searchsorted(ub // ns, np.arange(npt + 1))
    lcol_b = (np.searchsorted(ub, tile_b * ns + hm.b_col) - offb[tile_b]).astype(np.int32)
    nvp = np.diff(offb)
    segsys_p = nvp * W2 * 8
    t_, id_, slot, ln = _runs(ub, ns, offb)
    for m in range(2):
        add(nvt + t_, 0, (m * N * J + id_ * W2) * 8, m * segsys_p[t_] + slot * W2 * 8, ln * W2 * 8, 0)
    cur = 2 * segsys_p
    b0, b1 = hm.b_rowptr[p0].astype(np.int64), hm.b_rowptr[p1].astype(np.int64)
    o_rp, cur = stream(pt, 2, 7, p0, p1 + 1, 4, cur)
    o_col, cur = stream(pt, 3, 8, b0, b1, 4, cur)
    o_bv, cur = stream(pt, 4, 9, b0, b1, 16, cur)
    assert np.array_equal(cur, psz), "pressure tile sizes disagree"
    desc[nvt:, 0] = 1
    desc[nvt:, 1], desc[nvt:, 2] = p0, p1
    desc[nvt:, 5] = cur
    desc[nvt:, 6], desc[nvt:, 7] = segsys_p, 0
    desc[nvt:, 8], desc[nvt:, 9], desc[nvt:, 10] = o_rp, o_col, o_bv
    # ---- records grouped per tile
    r = np.concatenate(recs).view(np.recarray)
    o = np.lexsort((r.order, r.tile))
    r = r[o]
    if (r.nb >= 1 << 24).any() or (r.nb % 16).any() or (r.dst % 16).any() or (r.src % 16).any():
        raise ValueError("SpMM tile copy records violate the 16-byte bulk-copy rules")
    out = np.zeros(len(r), REC_DTYPE)
    out["src"], out["dst"], out["bk"] = r.src, r.dst, r.nb | (r.kind << 24)
    roff = np.searchsorted(r.tile, np.arange(ntile + 1))
    desc[:, 3] = roff[:-1]
    desc[:, 4] = np.diff(roff)
    stage = int(_a16(desc[:, 5].max()))
    info = dict(nvt=nvt, npt=npt, nrec=len(out), stage_bytes=stage,
                staged_bytes=int(desc[:, 5].astype(np.int64).sum()),
                mean_rows_v=float(ns / nvt), mean_rows_p=float(npres / max(npt, 1)))
    return desc, out, lcol_a, lcol_bt, lcol_b, info


def emulate(hm, J, desc, recs, lcol_a, lcol_bt, lcol_b, as_vals, X, B=None, mode=0):
    """numpy execution of the tile schedule (same staging arithmetic as the kernel): CPU check of the tiling."""
    N = hm.ntot
    H = J // 2
    srcs = {0: X.reshape(-1).view(np.uint8), 1: as_vals.reshape(-1).view(np.uint8),
            2: hm.s_rowptr.view(np.uint8), 3: lcol_a.view(np.uint8), 4: hm.bt_rowptr.view(np.uint8),
            5: lcol_bt.view(np.uint8), 6: hm.bt_val.view(np.uint8), 7: hm.b_rowptr.view(np.uint8),
            8: lcol_b.view(np.uint8), 9: hm.b_val.view(np.uint8)}
    srcs = {k: np.concatenate([v, np.zeros(64, np.uint8)]) for k, v in srcs.items()}   # device arrays are padded
    Xv = X.reshape(2, N, J)
    Y = np.zeros_like(Xv)
    for d in desc:
        st = np.zeros(int(d[5]) + 64, np.uint8)
        for rc in recs[d[3]:d[3] + d[4]]:
            kind, nb = int(rc["bk"]) >> 24, int(rc["bk"]) & 0xFFFFFF
            st[rc["dst"]:rc["dst"] + nb] = srcs[kind][rc["src"]:rc["src"] + nb]

        def rd(o, k, dt):
            it = np.dtype(dt).itemsize
            return st[o + k * it:o + (k + 1) * it].view(dt)[0]

        seg1 = int(d[6])
        if d[0] == 0:
            for node in range(d[1], d[2]):
                acc = np.zeros((2, 2 * J))
                for k in range(rd(d[8], node, np.int32), rd(d[8], node + 1, np.int32)):
                    lc = rd(d[9], k, np.int32)
                    a = (rd(d[10], k, np.float64), rd(d[11], k, np.float64))
                    for m in range(2):
                        o = m * seg1 + lc * 2 * J * 8
                        acc[m] += a[m] * st[o:o + 2 * J * 8].view(np.float64)
                for q in range(rd(d[12], node, np.int32), rd(d[12], node + 1, np.int32)):
                    lq = rd(d[13], q, np.int32)
                    bxy = st[d[14] + 16 * q:d[14] + 16 * q + 16].view(np.float64)
                    for m in range(2):
                        o = m * seg1 + d[7] + lq * J * 8
                        xp = st[o:o + J * 8].view(np.float64)
                        acc[m, :J] -= bxy[0] * xp
                        acc[m, J:] -= bxy[1] * xp
                for m in range(2):
                    rows = slice(2 * node * J, 2 * node * J + 2 * J)
                    Yr = Y[m].reshape(-1)[rows]
                    Yr[:] = acc[m]
                    for c in range(2):
                        if hm.cflag[2 * node + c]:
                            Yr[c * J:(c + 1) * J] = Xv[m].reshape(-1)[rows][c * J:(c + 1) * J]
                    Y[m].reshape(-1)[rows] = Yr
        else:
            for p in range(d[1], d[2]):
                acc = np.zeros((2, J))
                for q in range(rd(d[8], p, np.int32), rd(d[8], p + 1, np.int32)):
                    lc = rd(d[9], q, np.int32)
                    bxy = st[d[10] + 16 * q:d[10] + 16 * q + 16].view(np.float64)
                    for m in range(2):
                        o = m * seg1 + lc * 2 * J * 8
                        xs = st[o:o + 2 * J * 8].view(np.float64)
                        acc[m] += bxy[0] * xs[:J] + bxy[1] * xs[J:]
                row = hm.nvel + p
                for m in range(2):
                    Y[m, row] = Xv[m, row] if hm.cflag[row] else acc[m]
    if mode == 1:
        Y = B.reshape(2, N, J) - Y
    return Y


def _pair_union(row_ptr, cols, ncol, nrows):
    """Union of the column lists of rows 2p, 2p+1 (sorted), with each row's entry index or -1."""
    npair = (nrows + 1) // 2
    row_of = np.repeat(np.arange(nrows, dtype=np.int64), np.diff(row_ptr))
    k = np.arange(len(cols), dtype=np.int64)
    pair, h = row_of >> 1, row_of & 1
    key = pair * ncol + cols.astype(np.int64)
    o = np.lexsort((h, key))
    ukey, inv = np.unique(key[o], return_inverse=True)
    slots = np.full((len(ukey), 2), -1, dtype=np.int32)
    slots[inv, h[o]] = k[o]
    ptr = np.searchsorted(ukey // ncol, np.arange(npair + 1)).astype(np.int32)
    return ptr, (ukey % ncol).astype(np.int32), slots


def row_pairs(hm):
    """Row-pair structure of the velocity rows for the paired SpMM kernel (csrc/ens_spmm.cu)."""
    a = _pair_union(hm.s_rowptr, hm.s_col, hm.ns, hm.ns)
    t = _pair_union(hm.bt_rowptr, hm.bt_col, hm.npres, hm.ns)
    info = dict(npairs=(hm.ns + 1) // 2, a_union=len(a[1]), a_nnz=int(hm.nnz_s), t_union=len(t[1]),
                t_nnz=len(hm.bt_col))
    return a, t, info
