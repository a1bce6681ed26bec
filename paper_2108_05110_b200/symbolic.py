"""Symbolic analysis for the per-step saddle-point factorisation (host, once per mesh).

The reference factorises the assembled saddle matrix every sub-step with a
sparse direct LU (UMFPACK or SuperLU, `linalg.py:79-108`, called from
`stepper.py:216`) and solves all J columns with it (`linalg.py:62-76`).  The
B200 engine keeps that robustness but builds the factorisation on the GPU as
the *preconditioner* of a column-batched FGMRES: a multifrontal LU whose
symbolic structure is fixed per mesh (the pattern of the saddle matrix never
changes, `stepper.py:216-218`), computed here once.

Design:
  * Ordering: geometric nested dissection over the P2 nodes (one-sided vertex
    separators along mesh lines), giving an elimination tree of *fronts*.
  * Dof placement: a node's free velocity dofs go to the node's tree node; every
    free pressure dof is moved *up* to the highest tree node among its velocity
    neighbours, and inside each front velocities precede pressures.  With that
    order every leading principal block is a saddle system whose B rows are
    complete rows of the full B, hence nonsingular whenever the full matrix is
    (the velocity block is positive-real) -- LU without cross-panel pivoting is
    well defined.  Panels use partial pivoting internally (explicit inverse).
  * Dirichlet rows and the pressure pin are identity rows in the reference
    (`stepper.py:214-215`); they are eliminated trivially and never enter a
    front (the Krylov iterate carries their values exactly).
  * Each front's pivots are split into panels of <= PW dofs; the numeric phase
    sweeps them (block Gauss-Jordan) so a factorised front holds
    [-F11^-1, F11^-1 F12; F21 F11^-1, S] and every solve is one batched GEMM per
    tree level and direction (csrc/ens_mf.cu, csrc/ens_mfsolve.cu).

Everything returned is flat int32/int64 numpy arrays plus a launch schedule,
uploaded once by the engine.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

PW = 64          # panel width (max pivots per diagonal block)
TILE = 64        # GEMM tile edge in the numeric kernels
# tree heights (leaves = 0) whose nodes are merged into their parents (ENS_AMALG="1,3")
AMALGAMATE = tuple(int(x) for x in __import__("os").environ.get("ENS_AMALG", "1").split(",") if x.strip())
LEAF_NODES = int(__import__("os").environ.get("ENS_LEAF", "48"))  # stop dissecting below this many P2 nodes (48: a balanced tree, one level fewer than 24 at the same fill)


# ----------------------------------------------------------------------
# nested dissection on the P2 node graph
# ----------------------------------------------------------------------


_HOST = None


def _host():
    """ctypes handle on libensmhd_host.so (csrc/host_symbolic.cpp), built on first use."""
    global _HOST
    if _HOST is None:
        import ctypes as C
        from . import build as B
        lib = C.CDLL(B.build_host())
        P = C.c_void_p
        lib.ens_host_nested_dissection.restype = C.c_int64
        lib.ens_host_nested_dissection.argtypes = [C.c_int64, P, C.c_int64, P, P, C.c_int64, C.c_int64, P, P, P]
        lib.ens_host_symbolic_cb.restype = C.c_int64
        lib.ens_host_symbolic_cb.argtypes = [C.c_int64, P, P, P, P, P, P, P]
        lib.ens_host_front_local.restype = None
        lib.ens_host_front_local.argtypes = [C.c_int64, P, P, P, P, P]
        lib.ens_host_argsort_i64.restype = None
        lib.ens_host_argsort_i64.argtypes = [C.c_int64, P, P]
        lib.ens_host_sort_i64.restype = None
        lib.ens_host_sort_i64.argtypes = [C.c_int64, P]
        lib.ens_host_searchsorted_i64.restype = None
        lib.ens_host_searchsorted_i64.argtypes = [C.c_int64, P, C.c_int64, P, P]
        _HOST = lib
    return _HOST


def _ptr(a):
    return a.ctypes.data


def host_argsort(keys):
    """np.argsort(keys, kind="stable") for int64 keys, on all host cores (ens_host_argsort_i64)."""
    k = np.ascontiguousarray(keys, dtype=np.int64)
    out = np.empty(k.size, dtype=np.int64)
    _host().ens_host_argsort_i64(k.size, _ptr(k), _ptr(out))
    return out


def host_sort(keys):
    """np.sort(keys) for int64 keys (a new array), on all host cores (ens_host_sort_i64)."""
    k = np.array(keys, dtype=np.int64, copy=True, order="C")
    _host().ens_host_sort_i64(k.size, _ptr(k))
    return k


def host_searchsorted(a, q):
    """np.searchsorted(a, q) (left) for int64, on all host cores (ens_host_searchsorted_i64)."""
    a = np.ascontiguousarray(a, dtype=np.int64)
    q = np.ascontiguousarray(q, dtype=np.int64)
    out = np.empty(q.size, dtype=np.int64)
    _host().ens_host_searchsorted_i64(a.size, _ptr(a), q.size, _ptr(q), _ptr(out))
    return out


def _nested_dissection(coords, indptr, indices, leaf=LEAF_NODES):
    """Return (tree_nodes: list of node arrays, children: list of lists, root).

    Runs csrc/host_symbolic.cpp (ens_host_nested_dissection), the C++ restatement of
    `_nested_dissection_py` below (which remains the specification)."""
    n = coords.shape[0]
    rows = np.ascontiguousarray(np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr)))
    cols = np.ascontiguousarray(indices, dtype=np.int64)
    xy = np.ascontiguousarray(coords, dtype=np.float64)
    cap = 2 * n + 16
    off = np.zeros(cap + 1, dtype=np.int64)
    nodes = np.zeros(n, dtype=np.int64)
    par = np.zeros(cap, dtype=np.int64)
    T = _host().ens_host_nested_dissection(n, _ptr(xy), len(rows), _ptr(rows), _ptr(cols), int(leaf), cap,
                                           _ptr(off), _ptr(nodes), _ptr(par))
    if T < 0:
        raise RuntimeError("nested dissection: tree capacity exceeded")
    tnodes = [nodes[off[t]:off[t + 1]].copy() for t in range(T)]
    kids = [[] for _ in range(T)]
    for t in range(1, T):
        kids[par[t]].append(t)
    return tnodes, kids, 0


def _nested_dissection_py(coords, indptr, indices, leaf=LEAF_NODES):
    """Return (tree_nodes: list of node arrays, children: list of lists, root)."""
    n = coords.shape[0]
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    cols = indices.astype(np.int64)
    tnodes, kids = [], []

    # iterative (explicit stack) to avoid recursion limits on big meshes; every
    # subproblem carries its own edge list (edges with both ends inside it), so a
    # tree level costs O(nnz) instead of O(nnz) per tree node
    side = np.zeros(n, dtype=np.int8)
    stack = [(np.arange(n, dtype=np.int64), rows, cols, -1)]
    while stack:
        idx, er, ec, parent = stack.pop()
        me = len(tnodes)
        tnodes.append(None)
        kids.append([])
        if parent >= 0:
            kids[parent].append(me)
        if len(idx) <= leaf:
            tnodes[me] = idx
            continue
        c = coords[idx]
        ax = int(np.argmax(c.max(0) - c.min(0)))
        xs = c[:, ax]
        vals = np.unique(xs)
        med = np.sort(xs)[len(xs) // 2]
        ci = int(np.searchsorted(vals, med))
        xr, xc = coords[er, ax], coords[ec, ax]
        best = None
        for cut in vals[max(0, ci - 4):ci + 5]:
            nleft = int(np.count_nonzero(xs <= cut))
            nright = len(idx) - nleft
            if nleft == 0 or nright == 0:
                continue
            sep = np.unique(er[(xr <= cut) & (xc > cut)])
            bal = min(nleft - len(sep), nright) / len(idx)
            if bal < 0.25:
                continue
            score = len(sep) * (1.0 + 2.0 * abs(0.5 - bal))
            if best is None or score < best[0]:
                best = (score, cut, sep)
        if best is None:
            tnodes[me] = idx
            continue
        _, cut, sep = best
        side[idx] = np.where(xs > cut, 2, 1)
        side[sep] = 0
        sidx = side[idx]
        left = idx[sidx == 1]
        right = idx[sidx == 2]
        tnodes[me] = sep
        sr, sc = side[er], side[ec]
        for part, code in ((right, 2), (left, 1)):
            if len(part):
                keep = (sr == code) & (sc == code)
                stack.append((part, er[keep], ec[keep], me))
    return tnodes, kids, 0


def _amalgamate(tnodes, kids, root, heights):
    """Merge every tree node whose height (leaves = 0) is in `heights` into its parent: the parent's
    front then eliminates both separators (more fill, one tree level -- one launch round of every
    sweep -- fewer).  Returns (tnodes, kids, root) of the reduced tree."""
    if not heights:
        return tnodes, kids, root
    T = len(tnodes)
    order = _postorder(kids, root)
    height = np.zeros(T, dtype=np.int64)
    parent = np.full(T, -1, dtype=np.int64)
    for t in order:
        for c in kids[t]:
            parent[c] = t
            height[t] = max(height[t], height[c] + 1)
    gone = np.zeros(T, dtype=bool)
    nodes = [np.asarray(x) for x in tnodes]
    kk = [list(k) for k in kids]
    for t in order:   # children before parents: a merged node's kids are final when it is merged
        if t == root or height[t] not in heights:
            continue
        p = parent[t]
        nodes[p] = np.concatenate([nodes[t], nodes[p]])
        kk[p] = [c for c in kk[p] if c != t] + kk[t]
        for c in kk[t]:
            parent[c] = p
        gone[t] = True
    new_id = np.cumsum(~gone) - 1
    keep = [t for t in range(T) if not gone[t]]
    return ([nodes[t] for t in keep], [[int(new_id[c]) for c in kk[t]] for t in keep], int(new_id[root]))


def _postorder(kids, root):
    out, stack = [], [(root, False)]
    while stack:
        u, done = stack.pop()
        if done:
            out.append(u)
            continue
        stack.append((u, True))
        for c in reversed(kids[u]):
            stack.append((c, False))
    return np.array(out, dtype=np.int64)


@dataclass
class FactorPlan:
    """Everything the device factorisation / triangular solves need."""

    # internal numbering
    node_perm: np.ndarray        # P2 node (reference numbering) -> internal node id
    pres_perm: np.ndarray        # pressure dof -> internal pressure index (0..n_pres)
    # fronts (in processing order: by level, then position)
    nfront: int
    f_m: np.ndarray              # int32 front size
    f_k: np.ndarray              # int32 pivots
    f_off: np.ndarray            # int64 offset of the dense m x m front (per matrix)
    f_idx_off: np.ndarray        # int64 offset into f_idx
    f_idx: np.ndarray            # int32 internal dof ids of the front rows ([pivots; CB])
    f_level: np.ndarray
    f_parent: np.ndarray         # front id of the parent (-1 root)
    f_cmap_off: np.ndarray       # int64 offset of this front's CB -> parent-local map
    f_cmap: np.ndarray           # int32
    front_storage: int           # doubles per matrix
    # original entries -> front slots
    orig_dst: np.ndarray         # int64 slot (per matrix storage)
    orig_src: np.ndarray         # int32: < nnz_s -> A_s value; else signed B value index + nnz_s
    orig_level_off: np.ndarray   # int64 per level range in orig_*
    bsrc_vals: np.ndarray        # float64 constant (signed) B / -B^T values
    nlevels: int
    level_front_off: np.ndarray  # int32 fronts of level L are [off[L], off[L+1])
    level_storage_off: np.ndarray  # int64 storage range of level L
    schedule: dict               # launch work lists (see build_schedule)
    stats: dict


_TRACE = __import__("os").environ.get("ENS_SETUP_TRACE") == "1"


class _Tick:
    """Phase timer of analyse() (ENS_SETUP_TRACE=1 prints one line per phase)."""

    def __init__(self):
        import time
        self.clock, self.t = time.perf_counter, time.perf_counter()

    def __call__(self, label):
        if _TRACE:
            now = self.clock()
            print(f"  analyse: {label:28s} {now - self.t:7.3f} s", flush=True)
            self.t = now


def analyse(disc, leaf=LEAF_NODES, pw=PW):
    """Build the FactorPlan for a Discretization (constrained rows per disc)."""
    tick = _Tick()
    vel = disc.velocity
    ns, nvel, npres = disc.n_scalar, disc.n_vel, disc.n_pres
    n_total = nvel + npres
    from . import fe
    pat = fe.scalar_pattern(vel)
    g = pat.copy()
    g.setdiag(0)
    g.eliminate_zeros()
    g.sort_indices()
    tick("pattern")
    tnodes, kids, root = _nested_dissection(vel.dof_coords, g.indptr, g.indices, leaf)
    tnodes, kids, root = _amalgamate(tnodes, kids, root, AMALGAMATE)
    tick("dissection + amalgamation")
    post = _postorder(kids, root)
    T = len(tnodes)
    rank = np.empty(T, dtype=np.int64)
    rank[post] = np.arange(T)

    # internal node numbering: tree nodes in postorder, nodes in coordinate order inside
    # (vectorised over tree nodes: inside a tree node, nodes are sorted along the node's main axis,
    # then the other coordinate, then their position in the tree node -- SpMM locality)
    coords = vel.dof_coords
    sizes = np.array([len(tnodes[t]) for t in post], dtype=np.int64)
    cat = np.concatenate([tnodes[t] for t in post]).astype(np.int64)
    grp = np.repeat(np.arange(T, dtype=np.int64), sizes)
    within = np.arange(len(cat), dtype=np.int64) - np.repeat(np.cumsum(sizes) - sizes, sizes)
    cc = coords[cat]
    starts = np.cumsum(sizes) - sizes
    nz = sizes > 0
    ext = np.zeros((T, 2))
    ext[nz] = np.maximum.reduceat(cc, starts[nz], axis=0) - np.minimum.reduceat(cc, starts[nz], axis=0)
    ax_t = np.where(ext[:, 1] > ext[:, 0], 1, 0)
    ax_n = ax_t[grp]
    multi = sizes[grp] > 1
    prim = np.where(multi, cc[np.arange(len(cat)), ax_n], 0.0)
    sec = np.where(multi, cc[np.arange(len(cat)), 1 - ax_n], 0.0)
    o = np.lexsort((within, sec, prim, grp))
    node_perm = np.empty(ns, dtype=np.int64)
    node_perm[cat[o]] = np.arange(len(cat))
    tnode_of_node = np.empty(ns, dtype=np.int64)
    tnode_of_node[cat] = post[grp]

    tick("node numbering")
    # free dofs (reference numbering): velocity x = s, y = ns + s ; pressure nvel + p
    cons = np.zeros(n_total, dtype=bool)
    cons[disc.constrained_rows] = True

    # pressure placement: highest (max postorder rank) tree node over its velocity neighbours
    B = disc.divergence.tocsr()
    bnodes = B.indices % ns
    brow = np.repeat(np.arange(npres), np.diff(B.indptr))
    pres_node = disc.pressure.node_of_dof(vel)
    cand_rank = rank[tnode_of_node[bnodes]]
    best = np.full(npres, -1, dtype=np.int64)
    np.maximum.at(best, brow, cand_rank)
    best = np.maximum(best, rank[tnode_of_node[pres_node]])
    tnode_of_pres = post[best]

    # pressure internal order: by tree rank, then by the reference index
    # within a tree node, pressures are ordered along the node group's main axis
    # (moved-up pressures from both sides of a separator interleave spatially)
    pc = disc.pressure.dof_coords
    grp_order = np.argsort(best, kind="stable")
    bounds = np.searchsorted(best[grp_order], np.unique(best))
    gsz = np.diff(np.append(bounds, npres))
    pcs = pc[grp_order]
    gext = np.maximum.reduceat(pcs, bounds, axis=0) - np.minimum.reduceat(pcs, bounds, axis=0)
    gax = np.where((gsz > 1) & (gext[:, 1] > gext[:, 0]), 1, 0)
    axp = np.repeat(gax, gsz)
    key2 = np.empty(npres)
    key2[grp_order] = pcs[np.arange(npres), axp] * 4.0 + pcs[np.arange(npres), 1 - axp] * 1e-6
    porder = np.lexsort((np.arange(npres), key2, best))
    pres_perm = np.empty(npres, dtype=np.int64)
    pres_perm[porder] = np.arange(npres)

    tick("pressure placement")
    # internal dof id of every reference dof
    int_id = np.empty(n_total, dtype=np.int64)
    int_id[:ns] = 2 * node_perm
    int_id[ns:nvel] = 2 * node_perm + 1
    int_id[nvel:] = nvel + pres_perm

    # elimination order of free dofs: tree rank, then velocities before pressures, then internal id
    dof_t = np.empty(n_total, dtype=np.int64)
    dof_t[:ns] = tnode_of_node
    dof_t[ns:nvel] = tnode_of_node
    dof_t[nvel:] = tnode_of_pres
    is_p = np.zeros(n_total, dtype=np.int64)
    is_p[nvel:] = 1
    free = np.nonzero(~cons)[0]
    order = free[np.lexsort((int_id[free], is_p[free], rank[dof_t[free]]))]
    nf = len(order)
    elim = np.full(n_total, -1, dtype=np.int64)
    elim[order] = np.arange(nf)

    tick("elimination order")
    # free saddle pattern in elimination order (symmetric structure): the stored entries of
    # [[A_s, 0, Bx^T], [0, A_s, By^T], [Bx, By, 0]] + its transpose (a B entry that is exactly
    # zero cancels out of that sum and is not in the pattern), between free dofs, as CSR with
    # sorted rows
    As = pat.tocsr()
    a_r = np.repeat(np.arange(ns, dtype=np.int64), np.diff(As.indptr))
    a_c = As.indices.astype(np.int64)
    b_r = np.repeat(np.arange(npres, dtype=np.int64), np.diff(B.indptr))[B.data != 0.0] + nvel
    b_c = B.indices.astype(np.int64)[B.data != 0.0]
    pr_ = np.concatenate([a_r, a_r + ns, b_r, b_c])
    pc_ = np.concatenate([a_c, a_c + ns, b_c, b_r])
    pr_, pc_ = elim[pr_], elim[pc_]
    keep_ = (pr_ >= 0) & (pc_ >= 0)
    pkey = host_sort(pr_[keep_] * nf + pc_[keep_])
    fp = sp.csr_matrix((np.ones(pkey.size), (pkey % nf).astype(np.int32),
                        np.concatenate([[0], np.cumsum(np.bincount(pkey // nf, minlength=nf))])), shape=(nf, nf))
    del pr_, pc_, keep_, pkey, a_r, a_c, b_r, b_c

    tick("free pattern")
    # tree nodes -> pivot ranges in elimination order; drop empty tree nodes
    t_of_e = rank[dof_t[order]]                      # postorder rank per eliminated dof
    piv_start = np.searchsorted(t_of_e, np.arange(T), side="left")
    piv_end = np.searchsorted(t_of_e, np.arange(T), side="right")
    parent_r = np.full(T, -1, dtype=np.int64)        # by postorder rank
    for t in range(T):
        for c in kids[t]:
            parent_r[rank[c]] = rank[t]
    nonempty = piv_end > piv_start
    # re-parent through empty nodes
    eff_parent = parent_r.copy()
    for r in range(T):
        p = eff_parent[r]
        while p >= 0 and not nonempty[p]:
            p = parent_r[p]
        eff_parent[r] = p
    keep = np.nonzero(nonempty)[0]                   # ranks, increasing == postorder
    newid = np.full(T, -1, dtype=np.int64)
    newid[keep] = np.arange(len(keep))
    F = len(keep)
    fparent = np.where(eff_parent[keep] >= 0, newid[np.maximum(eff_parent[keep], 0)], -1)
    fparent[eff_parent[keep] < 0] = -1
    fs, fe_ = piv_start[keep], piv_end[keep]
    children = [[] for _ in range(F)]
    for f in range(F):
        if fparent[f] >= 0:
            children[fparent[f]].append(f)

    tick("tree bookkeeping")
    # symbolic factorisation: CB(f) = (later neighbours of pivots U children CBs) \ pivots, postorder
    # (children first); csrc/host_symbolic.cpp ens_host_symbolic_cb, the C++ restatement of
    #   cols = fp.indices[fp.indptr[s]:fp.indptr[e]];  cb[f] = unique(cols[cols >= e] U cb[c][cb[c] >= e])
    fs64, fe64 = np.ascontiguousarray(fs, dtype=np.int64), np.ascontiguousarray(fe_, dtype=np.int64)
    fpar64 = np.ascontiguousarray(fparent, dtype=np.int64)
    ip64 = np.ascontiguousarray(fp.indptr, dtype=np.int64)
    ind32 = np.ascontiguousarray(fp.indices, dtype=np.int32)
    cb_off = np.zeros(F + 1, dtype=np.int64)
    lib = _host()
    tot = lib.ens_host_symbolic_cb(F, _ptr(fs64), _ptr(fe64), _ptr(fpar64), _ptr(ip64), _ptr(ind32), _ptr(cb_off), None)
    cb_all = np.zeros(max(int(tot), 1), dtype=np.int64)
    lib.ens_host_symbolic_cb(F, _ptr(fs64), _ptr(fe64), _ptr(fpar64), _ptr(ip64), _ptr(ind32), _ptr(cb_off),
                             _ptr(cb_all))
    cb = [cb_all[cb_off[f]:cb_off[f + 1]] for f in range(F)]
    k = (fe_ - fs).astype(np.int64)
    cbn = np.array([len(c) for c in cb], dtype=np.int64)
    m = k + cbn

    tick("symbolic factorisation")
    # levels (height from leaves) -> processing order
    height = np.zeros(F, dtype=np.int64)
    for f in range(F):
        for c in children[f]:
            height[f] = max(height[f], height[c] + 1)
    nlevels = int(height.max()) + 1
    porder_f = np.lexsort((np.arange(F), height))    # processing order
    pid = np.empty(F, dtype=np.int64)
    pid[porder_f] = np.arange(F)
    level_front_off = np.searchsorted(height[porder_f], np.arange(nlevels + 1)).astype(np.int32)

    f_m = m[porder_f]
    f_k = k[porder_f]
    f_level = height[porder_f]
    f_parent = np.where(fparent[porder_f] >= 0, pid[np.maximum(fparent[porder_f], 0)], -1)
    f_off = np.concatenate([[0], np.cumsum(f_m * f_m)]).astype(np.int64)
    storage = int(f_off[-1])
    f_off = f_off[:-1]
    level_storage_off = np.concatenate([f_off[level_front_off[:-1]], [storage]]).astype(np.int64)

    # front index lists in elimination positions, then internal dof ids
    elim_to_int = int_id[order]
    lists = []
    for f in porder_f:
        lists.append(np.concatenate([np.arange(fs[f], fe_[f]), cb[f]]))
    f_idx_off = np.concatenate([[0], np.cumsum(f_m)]).astype(np.int64)
    f_idx_elim = np.concatenate(lists)
    f_idx = elim_to_int[f_idx_elim].astype(np.int32)

    # local position of an elimination index in a front: every front's index list is ascending
    # (pivot range, then the sorted contribution block) -> binary search per query (C++)
    f_idx_elim = np.ascontiguousarray(f_idx_elim, dtype=np.int64)
    f_idx_off = np.ascontiguousarray(f_idx_off, dtype=np.int64)

    def lookup(front, epos):
        fq = np.ascontiguousarray(front, dtype=np.int64)
        eq = np.ascontiguousarray(epos, dtype=np.int64)
        out = np.empty(len(fq), dtype=np.int64)
        _host().ens_host_front_local(len(fq), _ptr(fq), _ptr(eq), _ptr(f_idx_off), _ptr(f_idx_elim), _ptr(out))
        assert np.all(out >= 0), "symbolic lookup failed"
        return out

    tick("levels + index lists")
    # child CB -> parent local map (all fronts in one lookup: positions in front order)
    pos_front = np.repeat(np.arange(F, dtype=np.int64), f_m)
    pos_local = np.arange(len(f_idx_elim), dtype=np.int64) - np.repeat(f_idx_off[:-1], f_m)
    is_cb = pos_local >= f_k[pos_front]
    assert np.all(f_parent[pos_front[is_cb]] >= 0), "root front must have an empty CB"
    f_cmap = lookup(f_parent[pos_front[is_cb]], f_idx_elim[is_cb]).astype(np.int32)
    cmap_off = np.concatenate([[0], np.cumsum(f_m - f_k)]).astype(np.int64)

    tick("child maps")
    # original entries: A_s (both components) and B / -B^T, between free dofs
    nnz_s = As.nnz
    a_rows = np.repeat(np.arange(ns), np.diff(As.indptr))
    a_cols = As.indices
    src_l, r_l, c_l = [], [], []
    for comp in range(2):
        r = comp * ns + a_rows
        c = comp * ns + a_cols
        src_l.append(np.arange(nnz_s, dtype=np.int64))
        r_l.append(r)
        c_l.append(c)
    b_rows = np.repeat(np.arange(npres), np.diff(B.indptr))
    b_cols = B.indices                                # 0..2ns
    nb = B.nnz
    bsrc_vals = np.concatenate([B.data, -B.data])
    # B entries: row nvel+p, col b_cols ; -B^T entries: row b_cols, col nvel+p
    src_l += [nnz_s + np.arange(nb), nnz_s + nb + np.arange(nb)]
    r_l += [nvel + b_rows, b_cols]
    c_l += [b_cols, nvel + b_rows]
    src = np.concatenate(src_l)
    rr = np.concatenate(r_l)
    cc = np.concatenate(c_l)
    ok = (~cons[rr]) & (~cons[cc])
    src, rr, cc = src[ok], rr[ok], cc[ok]
    er, ec = elim[rr], elim[cc]
    first = np.minimum(er, ec)
    # front owning elimination position `first`
    piv_front_of_e = np.empty(nf, dtype=np.int64)
    piv_front_of_e[f_idx_elim[~is_cb]] = pos_front[~is_cb]
    fr = piv_front_of_e[first]
    lr = lookup(fr, er)
    lc = lookup(fr, ec)
    dst = f_off[fr] + lr * f_m[fr] + lc
    o = host_argsort(dst)        # == lexsort((dst, level)): dst is unique and grows with the level
    orig_dst = dst[o].astype(np.int64)
    orig_src = src[o].astype(np.int32)
    orig_level_off = np.searchsorted(f_level[fr][o], np.arange(nlevels + 1)).astype(np.int64)

    tick("original-entry scatter")
    plan = FactorPlan(
        node_perm=node_perm, pres_perm=pres_perm, nfront=F,
        f_m=f_m.astype(np.int32), f_k=f_k.astype(np.int32), f_off=f_off,
        f_idx_off=f_idx_off, f_idx=f_idx, f_level=f_level.astype(np.int32), f_parent=f_parent.astype(np.int32),
        f_cmap_off=cmap_off, f_cmap=f_cmap, front_storage=storage,
        orig_dst=orig_dst, orig_src=orig_src, orig_level_off=orig_level_off, bsrc_vals=bsrc_vals,
        nlevels=nlevels, level_front_off=level_front_off, level_storage_off=level_storage_off,
        schedule={}, stats={},
    )
    plan.schedule = build_schedule(plan, pw)
    tick("schedule")
    # sweep flops: sum_{t<k} 2 (m - 1 - t)^2 = 2 (S(m - 1) - S(m - k - 1)), S(n) = n (n + 1) (2n + 1) / 6
    def sq_sum(n):
        n = n.astype(np.float64)
        return n * (n + 1.0) * (2.0 * n + 1.0) / 6.0
    flops = float(np.sum(2.0 * (sq_sum(f_m - 1) - sq_sum(f_m - f_k - 1))))
    plan.stats = dict(fronts=F, levels=nlevels, n_free=nf, max_m=int(f_m.max()), max_k=int(f_k.max()),
                      storage_doubles=storage, factor_flops=flops,
                      nnz_lu=float(np.sum(f_m.astype(np.float64) ** 2 - (f_m - f_k).astype(np.float64) ** 2)))
    return plan


# ----------------------------------------------------------------------
# launch schedule (work lists), consumed by csrc/mf.cu
# ----------------------------------------------------------------------

# op codes (must match csrc/mf.cu)
OP_ZERO, OP_ORIG, OP_EXTADD, OP_DIAG, OP_HPANEL, OP_UPDATE, OP_GPANEL = range(7)
SOP_FINIT, SOP_FEXT, SOP_FGEMM, SOP_BGATHER, SOP_BGEMM, SOP_FRED, SOP_BRED = range(7)
# inner length per solve-GEMM work item: 0 = chosen per level (see _choose_split),
# else a fixed length for every level (tests, experiments: ENS_SPLIT_K)
SPLIT_K = int(__import__("os").environ.get("ENS_SPLIT_K", "256"))
SPLIT_CANDIDATES = (64, 128, 192, 256)   # <= the solve kernel's SG_KMAX
# per-level launch model of the solve GEMM (measured on B200 at C2): resident CTAs,
# fixed CTA latency, per-32-column chunk time, extra latency of a split group's reduction
_SLOTS, _T0, _TCHUNK, _TRED = 3 * 148, 3.5, 1.1, 3.0


def _choose_split(Ks, rows):
    """Inner split minimising waves x CTA latency for one level (both systems)."""
    if SPLIT_K > 0:
        return SPLIT_K
    best, best_t = SPLIT_CANDIDATES[-1], None
    kmax = max(Ks) if len(Ks) else 1
    for s_ in SPLIT_CANDIDATES:
        ncta = 2 * sum(-(-r // SOLVE_ROWS) * max(1, -(-K // s_)) for K, r in zip(Ks, rows))
        waves = -(-ncta // _SLOTS)
        t = waves * (_T0 + _TCHUNK * -(-min(kmax, s_) // 32) + (_TRED if kmax > s_ else 0.0))
        if best_t is None or t < best_t - 1e-9:
            best, best_t = s_, t
    return best
MAX_GSRC = 4      # child contribution rows gathered per front-vector row
EXT_ROWS = 8      # child-CB rows per extend-add work item
VEC_ROWS = 64     # front-vector rows per init/gather/scatter work item
SOLVE_ROWS = 64   # rows per solve-GEMM work item (csrc/ens_mfsolve.cu SG_R)


def build_schedule(plan: FactorPlan, pw=PW):
    """Flat int32 work items + launch list for factorisation and solves.

    factor launches: (op, level, item_off, n_items, arg)
      OP_ZERO   level storage range is zeroed (memset)
      OP_ORIG   items = level's original-entry range (handled by index range)
      OP_EXTADD items (child, row0)              -- one launch per sibling rank
      OP_DIAG   items (front, a)                 -- a = panel start
      OP_HPANEL items (front, a, col0)
      OP_UPDATE items (front, a, row0, col0)
      OP_GPANEL items (front, a, row0)
    solve launches: (op, level, item_off, n_items, arg)
    """
    # (vectorised over fronts; the item order is the nested-loop order spelled out per op below)
    items = []
    nitems = [0]

    def add(cols):
        """Append work items given as equal-length int columns (padded to 4 with zeros)."""
        n = len(cols[0])
        arr = np.zeros((n, 4), np.int32)
        for j, c in enumerate(cols):
            arr[:, j] = c
        off = nitems[0]
        items.append(arr)
        nitems[0] += n
        return off, n

    def expand(counts):
        """(owner, k): owner i repeated counts[i] times, k = 0 .. counts[i] - 1."""
        counts = np.asarray(counts, dtype=np.int64)
        own = np.repeat(np.arange(len(counts), dtype=np.int64), counts)
        return own, np.arange(own.size, dtype=np.int64) - np.repeat(np.cumsum(counts) - counts, counts)

    F = plan.nfront
    fm, fk, lvl, par = (plan.f_m.astype(np.int64), plan.f_k.astype(np.int64), plan.f_level,
                        plan.f_parent.astype(np.int64))
    # children of a front in ascending order; a child's rank among its siblings
    cs = np.nonzero(par >= 0)[0]
    cs = cs[np.argsort(par[cs], kind="stable")]
    nkids = np.bincount(par[cs], minlength=F)
    sib_rank = np.full(F, -1, dtype=np.int64)
    sib_rank[cs] = expand(nkids)[1]
    cbn_all = fm - fk
    fl, sl = [], []
    for L in range(plan.nlevels):
        lo, hi = int(plan.level_front_off[L]), int(plan.level_front_off[L + 1])
        fl.append((OP_ZERO, L, 0, 0, 0))
        fl.append((OP_ORIG, L, 0, 0, 0))
        # extend-add by sibling rank r (conflict-free within a launch): for fronts f ascending,
        # child c = children[f][r], rows r0 = 0, EXT_ROWS, .. < |CB(c)|  -> items (c, r0)
        maxr = int(nkids[lo:hi].max()) if hi > lo else 0
        for r in range(maxr):
            c = cs[(sib_rank[cs] == r) & (par[cs] >= lo) & (par[cs] < hi)]   # ascending parent
            i, k = expand(-(-cbn_all[c] // EXT_ROWS))
            if i.size:
                off, n = add((c[i], k * EXT_ROWS))
                fl.append((OP_EXTADD, L, off, n, r))
        # block sweep (Gauss-Jordan) over the front's pivot panels; the update
        # covers every row/column outside the panel (index r' -> r' < a ? r' : r' + pw)
        fr = np.arange(lo, hi, dtype=np.int64)
        npan = int((-(-fk[fr] // pw)).max()) if hi > lo else 0
        for p in range(npan):
            a = p * pw
            act = fr[fk[fr] > a]
            t = fm[act] - np.minimum(pw, fk[act] - a)
            nt = -(-t // TILE)
            d = (act, np.full(act.size, a))                               # (f, a)
            i, k = expand(nt)                                             # f, then c0
            h = (act[i], np.full(i.size, a), k * TILE)                    # (f, a, c0); GPANEL (f, a, row0)
            i2, k2 = expand(nt * nt)                                      # f, then c0, then r0
            ntr = nt[i2]
            u = (act[i2], np.full(i2.size, a), (k2 % ntr) * TILE, (k2 // ntr) * TILE)   # (f, a, r0, c0)
            for op, cols in ((OP_DIAG, d), (OP_HPANEL, h), (OP_UPDATE, u), (OP_GPANEL, h)):
                if cols[0].size:
                    off, n = add(cols)
                    fl.append((op, L, off, n, p))
    # solve schedule: after the sweep a front holds [-F11^-1, F11^-1 F12; F21 F11^-1, S]
    #   forward  fr[k:m] -= F_CP fr[0:k]           (SOP_FGEMM, rows of the CB)
    #   backward x[piv]   = -[F_PP F_PC] [fr_P; x_C] (SOP_BGEMM, rows of the pivots)
    #   SOP_FINIT gathers a front's vector rows in one pass: b at the pivots plus
    #   the (<= MAX_GSRC) child contribution rows mapped onto each row (gsrc);
    #   SOP_BGEMM reads x[C] straight from the global iterate (no gather pass).
    #   Long inner dimensions are split (SPLIT_K) into independent work items that
    #   write partial products to scratch slots; SOP_*RED sums them in a fixed
    #   order (deterministic, no atomics) and applies the update.
    fwd, bwd = [], []
    nslot = [0]
    splits = []

    # Forward items gather their own inputs (b at the pivots + children's
    # contribution rows via gsrc), so there is no separate FINIT pass; a front
    # without a contribution block gets one pivot-only item (r0 = -1).  Split
    # items (slot >= 0) are reduced by the last-arriving CTA of their group.
    # The launch's 5th field is the largest inner range of its items; when a level
    # has split items it equals that level's split length (the kernels use it so).
    #   per front f (ascending): K = K_of(f), rws = rows_of(f), ns = max(1, ceil(K / split))
    #     pivot-only (rws == 0 and pivot_only): t0 = 0, SOLVE_ROWS, .. < K -> (f, -1 - t0, 0, -1)
    #     else r0 = 0, SOLVE_ROWS, .. < rws: ns == 1 -> (f, r0, 0, -1)
    #                                         else   -> (f, r0, ks, next free slot) for ks < ns
    def gemm_items(fronts, rws, K, pivot_only):
        split = _choose_split([int(x) for x in K], [max(1, int(x)) for x in rws]) if SPLIT_K <= 0 else SPLIT_K
        splits.append(split)
        nsplit = np.maximum(1, -(-K // split))
        piv = (rws == 0) & pivot_only
        cnt = np.where(piv, -(-K // SOLVE_ROWS), -(-rws // SOLVE_ROWS) * nsplit)
        i, k = expand(cnt)
        pi, ns_i = piv[i], nsplit[i]
        f_col = fronts[i]
        r0 = np.where(pi, -1 - k * SOLVE_ROWS, (k // ns_i) * SOLVE_ROWS)
        is_split = (~pi) & (ns_i > 1)
        ks = np.where(is_split, k % ns_i, 0)
        slot = np.where(is_split, nslot[0] + np.cumsum(is_split) - 1, -1)
        nslot[0] += int(is_split.sum())
        kk = np.minimum(K[~piv], split)
        kmax = max(1, int(kk.max())) if kk.size else 1
        return (f_col, r0, ks, slot), kmax

    for L in range(plan.nlevels):
        fronts = np.arange(plan.level_front_off[L], plan.level_front_off[L + 1], dtype=np.int64)
        g, kmax = gemm_items(fronts, fm[fronts] - fk[fronts], fk[fronts], True)
        off, n = add(g)
        fwd.append((SOP_FGEMM, L, off, n, kmax))
    for L in reversed(range(plan.nlevels)):
        fronts = np.arange(plan.level_front_off[L], plan.level_front_off[L + 1], dtype=np.int64)
        g, kmax = gemm_items(fronts, fk[fronts], fm[fronts], False)
        off, n = add(g)
        bwd.append((SOP_BGEMM, L, off, n, kmax))
    # gather sources: gsrc[row of front p] = absolute f_idx rows of child CB entries mapped there,
    # in slot order = (child ascending, CB row ascending)
    nidx = int(plan.f_idx_off[-1])
    gsrc = np.full((nidx, MAX_GSRC), -1, dtype=np.int64)
    ch = np.nonzero(par >= 0)[0]
    ncb = plan.f_cmap_off[ch + 1] - plan.f_cmap_off[ch]
    ci, crow = expand(ncb)
    c_of = ch[ci]
    dst = plan.f_idx_off[par[c_of]] + plan.f_cmap[plan.f_cmap_off[c_of] + crow]
    srcrow = plan.f_idx_off[c_of] + fk[c_of] + crow
    o = np.argsort(dst, kind="stable")
    slot = np.empty(dst.size, dtype=np.int64)
    _, first, cnt = np.unique(dst[o], return_index=True, return_counts=True)
    slot[o] = np.arange(dst.size) - np.repeat(first, cnt)
    assert np.all(slot < MAX_GSRC), "too many children contribute to one front row"
    gsrc[dst, slot] = srcrow
    assert nidx < 2 ** 31
    work = np.vstack(items) if items else np.zeros((0, 4), np.int32)
    return dict(work=np.ascontiguousarray(work.astype(np.int32)), gsrc=np.ascontiguousarray(gsrc.astype(np.int32)),
                nslot=int(nslot[0]), split_k=int(max(splits) if splits else 1), solve_rows=int(SOLVE_ROWS),
                factor=np.array(fl, dtype=np.int64).reshape(-1, 5),
                fwd=np.array(fwd, dtype=np.int64).reshape(-1, 5),
                bwd=np.array(bwd, dtype=np.int64).reshape(-1, 5))
