"""Tile schedule of the staged SpMM (spmm_tiles.py): numpy execution of the exact staging arithmetic
(copy records, stage origins, tile-local slots) against the assembled saddle operator, no GPU."""

import numpy as np
import pytest

from oracle import ensmhd_oracle as O
import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import spmm_tiles as T
from paper_2108_05110_b200.engine import host_mesh


@pytest.mark.parametrize("case,over,cap", [("C1", dict(n=8, J=4), 16 * 1024), ("C1", dict(n=6, J=10), 8 * 1024),
                                           ("C4", dict(k=1, J=6, length=6.0), 24 * 1024)])
def test_tiles_reproduce_saddle_product(case, over, cap, rng):
    disc, cfg, _ = P.build_case(case, **over)
    hm = host_mesh(disc)
    J = cfg.num_members
    desc, recs, la, lbt, lb, info = T.build_tiles(hm, J, cap=cap, rows0=16)
    assert info["stage_bytes"] <= cap and (desc[:, 5] % 16 == 0).all()
    x = rng.standard_normal((2, hm.ntot, J))
    b = rng.standard_normal((2, hm.ntot, J))
    a = rng.standard_normal((2, hm.nnz_s))
    y = T.emulate(hm, J, desc, recs, la, lbt, lb, a, x, b, mode=1)
    for m in range(2):
        # internal-order operator from the engine's own CSR arrays, checked against the oracle's saddle matrix
        vals = np.zeros(hm.nnz_s)
        vals[:] = a[m]
        K = O.saddle_matrix(hm_to_reference_block(hm, vals, disc), disc)
        xr = x[m][hm.int_id]
        ref = b[m][hm.int_id] - K @ xr
        assert np.max(np.abs(y[m][hm.int_id] - ref)) <= 1e-13 * np.abs(ref).max()


def hm_to_reference_block(hm, vals, disc):
    """A_s in the reference numbering from internal-order CSR values."""
    import scipy.sparse as sp
    rows = np.repeat(np.arange(hm.ns), np.diff(hm.s_rowptr))
    inv = np.empty(hm.ns, dtype=np.int64)
    inv[hm.plan.node_perm] = np.arange(hm.ns)
    return sp.csr_matrix((vals, (inv[rows], inv[hm.s_col])), shape=(hm.ns, hm.ns))


def test_tile_records_obey_bulk_copy_rules():
    disc, cfg, _ = P.build_case("C1", n=6, J=8)
    hm = host_mesh(disc)
    desc, recs, *_ = T.build_tiles(hm, cfg.num_members, cap=12 * 1024, rows0=32)
    nb = recs["bk"] & 0xFFFFFF
    assert (recs["src"] % 16 == 0).all() and (recs["dst"] % 16 == 0).all() and (nb % 16 == 0).all()
    for d in desc:   # every record stays inside its tile's stage, and the records fill it exactly once
        r = recs[d[3]:d[3] + d[4]]
        cover = np.zeros(d[5], np.int32)
        for rc, n in zip(r, nb[d[3]:d[3] + d[4]]):
            assert rc["dst"] + n <= d[5]
            cover[rc["dst"]:rc["dst"] + n] += 1
        assert cover.max() == 1 and nb[d[3]:d[3] + d[4]].sum() == d[5]
    with pytest.raises(ValueError):
        T.build_tiles(hm, 7)


@pytest.mark.parametrize("case,over", [("C1", dict(n=6, J=4)), ("C4", dict(k=1, J=6, length=6.0))])
def test_row_pairs_keep_each_rows_csr_order(case, over):
    """The paired SpMM's union lists hold, for each row of a pair, exactly its CSR entries in CSR order."""
    disc, cfg, _ = P.build_case(case, **over)
    hm = host_mesh(disc)
    (ap, ac, asl), (tp, tc, tsl), info = T.row_pairs(hm)
    assert info["a_union"] < info["a_nnz"] and info["t_union"] <= info["t_nnz"]
    for r in range(hm.ns):
        p, h = r >> 1, r & 1
        e = np.arange(ap[p], ap[p + 1])
        e = e[asl[e, h] >= 0]
        assert np.array_equal(asl[e, h], np.arange(hm.s_rowptr[r], hm.s_rowptr[r + 1]))
        assert np.array_equal(ac[e], hm.s_col[hm.s_rowptr[r]:hm.s_rowptr[r + 1]])
        e = np.arange(tp[p], tp[p + 1])
        e = e[tsl[e, h] >= 0]
        assert np.array_equal(tsl[e, h], np.arange(hm.bt_rowptr[r], hm.bt_rowptr[r + 1]))
        assert np.array_equal(tc[e], hm.bt_col[hm.bt_rowptr[r]:hm.bt_rowptr[r + 1]])
