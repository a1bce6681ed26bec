// Host-side symbolic analysis kernels of the multifrontal plan (symbolic.py), in C++.
//
// Setup runs once per mesh, but at BASELINE C5 (2.1M velocity dofs) the two
// per-tree-node loops of symbolic.py -- the geometric nested dissection and the
// symbolic factorisation (contribution-block index sets) -- took ~25 s of Python
// overhead.  Same algorithms, same results (node order,
// tie-breaking and floating-point comparisons mirror the Python definitions in
// symbolic.py, which remain the specification; tests/test_symbolic.py compares).
// Plain C ABI, loaded with ctypes; no CUDA.
#include <algorithm>
#include <cmath>
#include <cstdint>
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
// out_parent[t] (-1 root); tree nodes are numbered in creation order (children lists in that
// order).  Returns the number of tree nodes, or -1 if a capacity is too small.
int64_t ens_host_nested_dissection(int64_t n, const double* coords, int64_t ne, const int64_t* er0,
                                   const int64_t* ec0, int64_t leaf, int64_t cap_t, int64_t* out_off,
                                   int64_t* out_nodes, int64_t* out_parent) {
    std::vector<int8_t> side((size_t)n, 0);
    std::vector<Sub> stack;
    {
        Sub s;
        s.idx.resize((size_t)n);
        for (int64_t i = 0; i < n; ++i) s.idx[(size_t)i] = i;
        s.er.assign(er0, er0 + ne);
        s.ec.assign(ec0, ec0 + ne);
        s.parent = -1;
        stack.push_back(std::move(s));
    }
    int64_t T = 0, pos = 0;
    out_off[0] = 0;
    std::vector<double> xs, vals, xr, xc;
    while (!stack.empty()) {
        Sub cur = std::move(stack.back());
        stack.pop_back();
        const int64_t me = T++;
        if (me >= cap_t) return -1;
        out_parent[me] = cur.parent;
        const int64_t m = (int64_t)cur.idx.size();
        auto emit = [&](const std::vector<int64_t>& nodes) {
            for (int64_t v : nodes) out_nodes[pos++] = v;
            out_off[me + 1] = pos;
        };
        if (m <= leaf) {
            emit(cur.idx);
            continue;
        }
        double lo[2] = {INFINITY, INFINITY}, hi[2] = {-INFINITY, -INFINITY};
        for (int64_t v : cur.idx)
            for (int d = 0; d < 2; ++d) {
                lo[d] = std::min(lo[d], coords[2 * v + d]);
                hi[d] = std::max(hi[d], coords[2 * v + d]);
            }
        const int ax = (hi[1] - lo[1]) > (hi[0] - lo[0]) ? 1 : 0;   // np.argmax: first maximum
        xs.resize((size_t)m);
        for (int64_t i = 0; i < m; ++i) xs[(size_t)i] = coords[2 * cur.idx[(size_t)i] + ax];
        vals = xs;
        std::sort(vals.begin(), vals.end());
        const double med = vals[(size_t)(m / 2)];
        vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
        const int64_t ci = std::lower_bound(vals.begin(), vals.end(), med) - vals.begin();
        const int64_t nedge = (int64_t)cur.er.size();
        xr.resize((size_t)nedge);
        xc.resize((size_t)nedge);
        for (int64_t e = 0; e < nedge; ++e) {
            xr[(size_t)e] = coords[2 * cur.er[(size_t)e] + ax];
            xc[(size_t)e] = coords[2 * cur.ec[(size_t)e] + ax];
        }
        bool have = false;
        double best_score = 0.0, best_cut = 0.0;
        std::vector<int64_t> best_sep, sep;
        const int64_t c0 = std::max<int64_t>(0, ci - 4), c1 = std::min<int64_t>((int64_t)vals.size(), ci + 5);
        for (int64_t q = c0; q < c1; ++q) {
            const double cut = vals[(size_t)q];
            int64_t nleft = 0;
            for (double x : xs) nleft += x <= cut ? 1 : 0;
            const int64_t nright = m - nleft;
            if (nleft == 0 || nright == 0) continue;
            sep.clear();
            for (int64_t e = 0; e < nedge; ++e)
                if (xr[(size_t)e] <= cut && xc[(size_t)e] > cut) sep.push_back(cur.er[(size_t)e]);
            std::sort(sep.begin(), sep.end());
            sep.erase(std::unique(sep.begin(), sep.end()), sep.end());
            const double bal = (double)std::min(nleft - (int64_t)sep.size(), nright) / (double)m;
            if (bal < 0.25) continue;
            const double score = (double)sep.size() * (1.0 + 2.0 * std::fabs(0.5 - bal));
            if (!have || score < best_score) {
                have = true;
                best_score = score;
                best_cut = cut;
                best_sep = sep;
            }
        }
        if (!have) {
            emit(cur.idx);
            continue;
        }
        for (int64_t i = 0; i < m; ++i) side[(size_t)cur.idx[(size_t)i]] = xs[(size_t)i] > best_cut ? 2 : 1;
        for (int64_t v : best_sep) side[(size_t)v] = 0;
        emit(best_sep);
        Sub parts[2];   // [0] right (code 2), [1] left (code 1): pushed in that order, the left pops first
        for (int h = 0; h < 2; ++h) {
            const int8_t code = h == 0 ? 2 : 1;
            for (int64_t v : cur.idx)
                if (side[(size_t)v] == code) parts[h].idx.push_back(v);
            for (int64_t e = 0; e < nedge; ++e)
                if (side[(size_t)cur.er[(size_t)e]] == code && side[(size_t)cur.ec[(size_t)e]] == code) {
                    parts[h].er.push_back(cur.er[(size_t)e]);
                    parts[h].ec.push_back(cur.ec[(size_t)e]);
                }
            parts[h].parent = me;
        }
        for (int h = 0; h < 2; ++h)
            if (!parts[h].idx.empty()) stack.push_back(std::move(parts[h]));
    }
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
    for (int64_t q = 0; q < nq; ++q) {
        const int64_t f = front[q];
        const int64_t* a = idx_elim + idx_off[f];
        const int64_t* b = idx_elim + idx_off[f + 1];
        const int64_t* p = std::lower_bound(a, b, epos[q]);
        out[q] = (p != b && *p == epos[q]) ? (int64_t)(p - a) : -1;
    }
}

}  // extern "C"
