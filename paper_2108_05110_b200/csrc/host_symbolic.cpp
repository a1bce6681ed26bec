// Host-side symbolic analysis kernels of the multifrontal plan (symbolic.py), in C++.
//
// Setup runs once per mesh, but at BASELINE C5 (2.1M velocity dofs) the two
// per-tree-node loops of symbolic.py -- the geometric nested dissection and the
// symbolic factorisation (contribution-block index sets) -- took ~25 s of Python
// overhead.  Same algorithms, same results (node order,
// tie-breaking and floating-point comparisons mirror the Python definitions in
// symbolic.py, which remain the specification; tests/test_symbolic.py compares).
// Plain C ABI, loaded with ctypes; no CUDA.  OpenMP over the host cores; every parallel
// routine returns exactly what its sequential definition returns.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <parallel/algorithm>
#include <utility>
#include <vector>

namespace {

struct Sub {
    std::vector<int64_t> idx, er, ec;
    int64_t parent;
};

}  // namespace

extern "C" {

// Geometric nested dissection on the P2 node graph (symbolic._nested_dissection):
// coords (n x 2, row-major), directed edge list (er, ec) of the pattern without the diagonal,
// leaf size.  Outputs: tree node t's nodes are out_nodes[out_off[t] .. out_off[t+1]), its parent
// out_parent[t] (-1 root); tree nodes are numbered in creation order of the specification's
// depth-first stack (a separator, then its left subtree, then its right subtree: preorder).
// Returns the number of tree nodes, or -1 if a capacity is too small.
//
// Parallel (OpenMP) without changing the result: the two halves of a split are independent
// subtrees (tasks; each returns its own preorder list, concatenated in the specification's order),
// and the up-to-9 candidate cuts of one split are scored concurrently and chosen in order.

struct Tree {
    std::vector<int64_t> off{0}, nodes, parent;   // preorder; parent local (-1 = this subtree's root)
    void add(const std::vector<int64_t>& nd, int64_t par) {
        nodes.insert(nodes.end(), nd.begin(), nd.end());
        off.push_back((int64_t)nodes.size());
        parent.push_back(par);
    }
    void append(const Tree& t, int64_t par_of_root) {   // t's nodes follow, its root under par_of_root
        const int64_t base = (int64_t)parent.size(), nb = (int64_t)nodes.size();
        nodes.insert(nodes.end(), t.nodes.begin(), t.nodes.end());
        for (size_t i = 1; i < t.off.size(); ++i) off.push_back(nb + t.off[i]);
        for (int64_t p : t.parent) parent.push_back(p < 0 ? par_of_root : base + p);
    }
};

static const int64_t ND_TASK_MIN = 20000;    // subproblems at least this big run as tasks

static void nd_rec(Sub cur, const double* coords, int64_t leaf, std::vector<int8_t>& side, Tree& out) {
    const int64_t m = (int64_t)cur.idx.size();
    if (m <= leaf) {
        out.add(cur.idx, -1);
        return;
    }
    double lo[2] = {INFINITY, INFINITY}, hi[2] = {-INFINITY, -INFINITY};
    for (int64_t v : cur.idx)
        for (int d = 0; d < 2; ++d) {
            lo[d] = std::min(lo[d], coords[2 * v + d]);
            hi[d] = std::max(hi[d], coords[2 * v + d]);
        }
    const int ax = (hi[1] - lo[1]) > (hi[0] - lo[0]) ? 1 : 0;   // np.argmax: first maximum
    std::vector<double> xs((size_t)m);
    for (int64_t i = 0; i < m; ++i) xs[(size_t)i] = coords[2 * cur.idx[(size_t)i] + ax];
    // median = sorted(xs)[m / 2]; candidate cuts = the distinct values around it: up to 4 below,
    // the median, up to 4 above (the specification's unique(xs)[ci - 4 .. ci + 5))
    std::vector<double> tmp = xs;
    std::nth_element(tmp.begin(), tmp.begin() + m / 2, tmp.end());
    const double med = tmp[(size_t)(m / 2)];
    std::vector<double> below, above;          // 4 largest distinct < med, 4 smallest distinct > med
    for (double x : xs) {
        if (x < med) {
            if (std::find(below.begin(), below.end(), x) != below.end()) continue;
            if (below.size() < 4) below.push_back(x);
            else {
                auto mn = std::min_element(below.begin(), below.end());
                if (x > *mn) *mn = x;
            }
        } else if (x > med) {
            if (std::find(above.begin(), above.end(), x) != above.end()) continue;
            if (above.size() < 4) above.push_back(x);
            else {
                auto mx = std::max_element(above.begin(), above.end());
                if (x < *mx) *mx = x;
            }
        }
    }
    std::sort(below.begin(), below.end());
    std::sort(above.begin(), above.end());
    std::vector<double> cuts(below);
    cuts.push_back(med);
    cuts.insert(cuts.end(), above.begin(), above.end());
    const int64_t nedge = (int64_t)cur.er.size();
    const int nc = (int)cuts.size();
    std::vector<std::vector<int64_t>> seps((size_t)nc);
    std::vector<double> score((size_t)nc, -1.0);   // < 0: candidate rejected
    const bool big = m >= ND_TASK_MIN;
#pragma omp taskloop if (big) default(shared)
    for (int q = 0; q < nc; ++q) {
        const double cut = cuts[(size_t)q];
        int64_t nleft = 0;
        for (double x : xs) nleft += x <= cut ? 1 : 0;
        const int64_t nright = m - nleft;
        if (nleft == 0 || nright == 0) continue;
        std::vector<int64_t>& sep = seps[(size_t)q];
        for (int64_t e = 0; e < nedge; ++e)
            if (coords[2 * cur.er[(size_t)e] + ax] <= cut && coords[2 * cur.ec[(size_t)e] + ax] > cut)
                sep.push_back(cur.er[(size_t)e]);
        std::sort(sep.begin(), sep.end());
        sep.erase(std::unique(sep.begin(), sep.end()), sep.end());
        const double bal = (double)std::min(nleft - (int64_t)sep.size(), nright) / (double)m;
        if (bal < 0.25) continue;
        score[(size_t)q] = (double)sep.size() * (1.0 + 2.0 * std::fabs(0.5 - bal));
    }
    int best = -1;
    for (int q = 0; q < nc; ++q)
        if (score[(size_t)q] >= 0.0 && (best < 0 || score[(size_t)q] < score[(size_t)best])) best = q;
    if (best < 0) {
        out.add(cur.idx, -1);
        return;
    }
    const double best_cut = cuts[(size_t)best];
    const std::vector<int64_t>& best_sep = seps[(size_t)best];
    for (int64_t i = 0; i < m; ++i) side[(size_t)cur.idx[(size_t)i]] = xs[(size_t)i] > best_cut ? 2 : 1;
    for (int64_t v : best_sep) side[(size_t)v] = 0;
    out.add(best_sep, -1);
    Sub parts[2];   // [0] left (code 1), [1] right (code 2): preorder visits the left subtree first
    for (int h = 0; h < 2; ++h) {
        const int8_t code = h == 0 ? 1 : 2;
        for (int64_t v : cur.idx)
            if (side[(size_t)v] == code) parts[h].idx.push_back(v);
        for (int64_t e = 0; e < nedge; ++e)
            if (side[(size_t)cur.er[(size_t)e]] == code && side[(size_t)cur.ec[(size_t)e]] == code) {
                parts[h].er.push_back(cur.er[(size_t)e]);
                parts[h].ec.push_back(cur.ec[(size_t)e]);
            }
    }
    { Sub().idx.swap(cur.idx); std::vector<int64_t>().swap(cur.er); std::vector<int64_t>().swap(cur.ec); }
    xs.clear(); xs.shrink_to_fit(); tmp.clear(); tmp.shrink_to_fit(); seps.clear();
    Tree sub[2];
    for (int h = 0; h < 2; ++h) {
        if (parts[h].idx.empty()) continue;
        const bool spawn = (int64_t)parts[h].idx.size() >= ND_TASK_MIN;
        Sub* ph = &parts[h];
        Tree* th = &sub[h];
#pragma omp task if (spawn) default(none) firstprivate(ph, th, coords, leaf) shared(side)
        nd_rec(std::move(*ph), coords, leaf, side, *th);
    }
#pragma omp taskwait
    for (int h = 0; h < 2; ++h)
        if (!sub[h].parent.empty()) out.append(sub[h], 0);
}

int64_t ens_host_nested_dissection(int64_t n, const double* coords, int64_t ne, const int64_t* er0,
                                   const int64_t* ec0, int64_t leaf, int64_t cap_t, int64_t* out_off,
                                   int64_t* out_nodes, int64_t* out_parent) {
    std::vector<int8_t> side((size_t)n, 0);   // disjoint subtrees write disjoint entries
    Sub s;
    s.idx.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) s.idx[(size_t)i] = i;
    s.er.assign(er0, er0 + ne);
    s.ec.assign(ec0, ec0 + ne);
    s.parent = -1;
    Tree t;
#pragma omp parallel
#pragma omp single
    nd_rec(std::move(s), coords, leaf, side, t);
    const int64_t T = (int64_t)t.parent.size();
    if (T > cap_t) return -1;
    std::copy(t.off.begin(), t.off.end(), out_off);
    std::copy(t.nodes.begin(), t.nodes.end(), out_nodes);
    std::copy(t.parent.begin(), t.parent.end(), out_parent);
    return T;
}

// Symbolic factorisation (symbolic.analyse): fronts f = 0..F-1 in postorder with pivot ranges
// [fs, fe) of the elimination order and parents; the symmetric free pattern in elimination order
// (CSR indptr / indices, sorted rows).  CB(f) = sorted unique (later neighbours of the pivots U
// children's CB entries >= fe(f)).  Writes cb_off (F+1) and, when cb is non-null, the entries;
// returns the total CB size.
int64_t ens_host_symbolic_cb(int64_t F, const int64_t* fs, const int64_t* fe, const int64_t* parent,
                             const int64_t* indptr, const int32_t* indices, int64_t* cb_off, int64_t* cb) {
    std::vector<std::vector<int64_t>> kids((size_t)F);
    for (int64_t f = 0; f < F; ++f)
        if (parent[f] >= 0) kids[(size_t)parent[f]].push_back(f);
    std::vector<std::vector<int64_t>> sets((size_t)F);
    std::vector<int64_t> buf;
    cb_off[0] = 0;
    for (int64_t f = 0; f < F; ++f) {
        const int64_t s = fs[f], e = fe[f];
        buf.clear();
        for (int64_t k = indptr[s]; k < indptr[e]; ++k)
            if (indices[k] >= e) buf.push_back(indices[k]);
        for (int64_t c : kids[(size_t)f]) {
            for (int64_t v : sets[(size_t)c])
                if (v >= e) buf.push_back(v);
            std::vector<int64_t>().swap(sets[(size_t)c]);   // a child's set is read once, by its parent
        }
        std::sort(buf.begin(), buf.end());
        buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
        cb_off[f + 1] = cb_off[f] + (int64_t)buf.size();
        if (cb) std::copy(buf.begin(), buf.end(), cb + cb_off[f]);
        sets[(size_t)f] = buf;
    }
    return cb_off[F];
}

// Local position of elimination index epos[q] in front front[q]: the front's index list
// idx_elim[idx_off[f] .. idx_off[f+1]) is ascending (pivot range, then the contribution block), so
// a binary search per query.  out[q] = -1 when absent.  (symbolic.analyse's `lookup`.)
void ens_host_front_local(int64_t nq, const int64_t* front, const int64_t* epos, const int64_t* idx_off,
                          const int64_t* idx_elim, int64_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nq; ++q) {
        const int64_t f = front[q];
        const int64_t* a = idx_elim + idx_off[f];
        const int64_t* b = idx_elim + idx_off[f + 1];
        const int64_t* p = std::lower_bound(a, b, epos[q]);
        out[q] = (p != b && *p == epos[q]) ? (int64_t)(p - a) : -1;
    }
}

// Permutation sorting int64 keys ascending, ties by position (== np.argsort(keys, kind="stable")).
void ens_host_argsort_i64(int64_t n, const int64_t* keys, int64_t* perm) {
    std::vector<std::pair<int64_t, int64_t>> kv((size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) kv[(size_t)i] = {keys[i], i};
    __gnu_parallel::sort(kv.begin(), kv.end());   // (key, position) pairs are distinct: order is unique
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) perm[i] = kv[(size_t)i].second;
}

// keys sorted ascending in place (== np.sort).
void ens_host_sort_i64(int64_t n, int64_t* keys) { __gnu_parallel::sort(keys, keys + n); }

// out[q] = lower_bound position of queries[q] in the ascending array a (== np.searchsorted(a, q)).
void ens_host_searchsorted_i64(int64_t na, const int64_t* a, int64_t nq, const int64_t* queries, int64_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nq; ++q) out[q] = std::lower_bound(a, a + na, queries[q]) - a;
}

}  // extern "C"
