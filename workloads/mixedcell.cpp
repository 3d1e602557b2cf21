// mixedcell.cpp — fine mixed cells of lifted supports (workload preparation, not the method).
//
// The paper assumes the start points of the polyhedral homotopy are given.
// This tool computes them for the benchmark systems the standard way (Huber-Sturmfels):
// a mixed cell is one pair {a_k, a'_k} of S_k per equation with an inner normal (alpha, 1),
//   <a_k, alpha> + w(a_k) = <a'_k, alpha> + w(a'_k) = beta_k,   <b, alpha> + w(b) > beta_k (b other).
// Enumeration: lower edges of every lifted support, a pairwise compatibility table, then a
// depth-first search over the supports that keeps a node only if the partial system has a
// solution with a positive margin (a small LP, solved through its dual with a dense simplex).
// Leaves are verified directly (alpha solves the n equalities; every inequality holds).
//
// C ABI (ctypes, workloads/startsys.py):
//   int mc_cells(int n, const int64_t *off, const int32_t *exps, const double *lift,
//                int64_t max_cells, int32_t *pairs_out /*[max][n][2] global term ids*/,
//                double *alpha_out /*[max][n]*/, double *gap_out /*[max]*/, int64_t *stats);
//   returns the number of cells (or -1 on overflow of max_cells).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

struct Support {
    std::vector<std::vector<double>> a; // exponents
    std::vector<double> w;              // liftings
    std::vector<int> gid;               // global term ids
};

struct Edge {
    int p, q; // local indices
};

// max t  s.t.  M y <= b  (y free, dim D), via the dual  min b^T l, M^T l = c, l >= 0,
// c = e_{D-1}.  Dense two-phase simplex with Bland's rule.  Returns the optimum (primal t*),
// or -inf if infeasible.
double lp_max_last(const std::vector<double> &M, const std::vector<double> &b, int m, int D)
{
    // tableau: D rows (equalities M^T l = c) + objective; columns: m dual vars + D artificials + rhs
    const int cols = m + D + 1;
    std::vector<double> T((size_t)(D + 1) * cols, 0.0);
    auto at = [&](int r, int c) -> double & { return T[(size_t)r * cols + c]; };
    for (int r = 0; r < D; ++r) {
        double rhs = (r == D - 1) ? 1.0 : 0.0;
        double sgn = rhs < 0 ? -1.0 : 1.0;
        for (int j = 0; j < m; ++j) at(r, j) = sgn * M[(size_t)j * D + r];
        at(r, m + r) = 1.0;
        at(r, cols - 1) = sgn * rhs;
    }
    std::vector<int> basis(D);
    for (int r = 0; r < D; ++r) basis[r] = m + r;
    const double eps = 1e-11;
    auto run = [&](std::vector<double> &cost, int ncols_allowed) -> bool {
        // objective row: reduced costs for minimisation of cost^T x
        for (int it = 0; it < 5000; ++it) {
            // reduced cost d_j = cost_j - sum_r cost_{basis r} T[r][j]
            int enter = -1;
            for (int j = 0; j < ncols_allowed; ++j) {
                double d = cost[j];
                for (int r = 0; r < D; ++r) d -= cost[basis[r]] * at(r, j);
                if (d < -eps) { enter = j; break; } // Bland: first improving column
            }
            if (enter < 0) return true;
            int leave = -1;
            double best = INFINITY;
            for (int r = 0; r < D; ++r) {
                double v = at(r, enter);
                if (v > eps) {
                    double ratio = at(r, cols - 1) / v;
                    if (ratio < best - 1e-14 || (std::fabs(ratio - best) <= 1e-14 && leave >= 0 && basis[r] < basis[leave])) {
                        best = ratio;
                        leave = r;
                    }
                }
            }
            if (leave < 0) return false; // unbounded (dual) -> primal infeasible
            double pv = at(leave, enter);
            for (int j = 0; j < cols; ++j) at(leave, j) /= pv;
            for (int r = 0; r < D; ++r) {
                if (r == leave) continue;
                double f = at(r, enter);
                if (f != 0.0)
                    for (int j = 0; j < cols; ++j) at(r, j) -= f * at(leave, j);
            }
            basis[leave] = enter;
        }
        return true;
    };
    // phase 1: minimise the sum of artificials
    std::vector<double> c1(m + D, 0.0);
    for (int r = 0; r < D; ++r) c1[m + r] = 1.0;
    run(c1, m + D);
    double art = 0.0;
    for (int r = 0; r < D; ++r)
        if (basis[r] >= m) art += at(r, cols - 1);
    if (art > 1e-9) return -INFINITY; // dual infeasible -> primal unbounded above (cannot happen with the cap)
    // drive remaining artificials out of the basis where possible
    for (int r = 0; r < D; ++r) {
        if (basis[r] < m) continue;
        for (int j = 0; j < m; ++j) {
            if (std::fabs(at(r, j)) > 1e-9) {
                double pv = at(r, j);
                for (int jj = 0; jj < cols; ++jj) at(r, jj) /= pv;
                for (int rr = 0; rr < D; ++rr) {
                    if (rr == r) continue;
                    double f = at(rr, j);
                    if (f != 0.0)
                        for (int jj = 0; jj < cols; ++jj) at(rr, jj) -= f * at(r, jj);
                }
                basis[r] = j;
                break;
            }
        }
    }
    // phase 2: minimise b^T l over the dual variables only
    std::vector<double> c2(m + D, 1e30);
    for (int j = 0; j < m; ++j) c2[j] = b[j];
    for (int r = 0; r < D; ++r) c2[m + r] = 0.0; // artificials stuck at zero level
    if (!run(c2, m)) return -INFINITY;           // dual unbounded below -> primal infeasible
    double obj = 0.0;
    for (int r = 0; r < D; ++r)
        if (basis[r] < m) obj += b[basis[r]] * at(r, cols - 1);
    return obj;
}

// Reduce the k equality rows E alpha = r to alpha = a0 + N beta (Gaussian elimination in double;
// the rows are small integer vectors).  Returns false if the equalities are inconsistent or
// dependent.
bool nullspace(int n, const std::vector<std::vector<double>> &E, const std::vector<double> &r,
               std::vector<double> &a0, std::vector<double> &N, int &d)
{
    const int k = (int)E.size();
    std::vector<std::vector<double>> A(E);
    std::vector<double> rhs(r);
    std::vector<int> pivcol(k, -1);
    int row = 0;
    std::vector<int> free_cols;
    for (int c = 0; c < n && row < k; ++c) {
        int p = -1;
        double best = 1e-12;
        for (int i = row; i < k; ++i)
            if (std::fabs(A[i][c]) > best) { best = std::fabs(A[i][c]); p = i; }
        if (p < 0) { free_cols.push_back(c); continue; }
        std::swap(A[p], A[row]);
        std::swap(rhs[p], rhs[row]);
        double pv = A[row][c];
        for (int j = 0; j < n; ++j) A[row][j] /= pv;
        rhs[row] /= pv;
        for (int i = 0; i < k; ++i) {
            if (i == row) continue;
            double f = A[i][c];
            if (f != 0.0) {
                for (int j = 0; j < n; ++j) A[i][j] -= f * A[row][j];
                rhs[i] -= f * rhs[row];
            }
        }
        pivcol[row] = c;
        ++row;
    }
    if (row < k) return false; // dependent rows
    for (int c = 0; c < n; ++c) {
        bool piv = false;
        for (int i = 0; i < k; ++i) piv |= (pivcol[i] == c);
        if (!piv && std::find(free_cols.begin(), free_cols.end(), c) == free_cols.end()) free_cols.push_back(c);
    }
    std::sort(free_cols.begin(), free_cols.end());
    d = (int)free_cols.size();
    a0.assign(n, 0.0);
    for (int i = 0; i < k; ++i) a0[pivcol[i]] = rhs[i];
    N.assign((size_t)n * d, 0.0);
    for (int f = 0; f < d; ++f) {
        int c = free_cols[f];
        N[(size_t)c * d + f] = 1.0;
        for (int i = 0; i < k; ++i) N[(size_t)pivcol[i] * d + f] = -A[i][c];
    }
    return true;
}

struct Solver {
    int n;
    std::vector<Support> S;
    std::vector<std::vector<Edge>> edges;
    int64_t lps = 0, nodes = 0;

    // margin of the chosen edges: max t such that some alpha satisfies the equalities and every
    // inequality of the involved supports with slack >= t (t capped at 1)
    double margin(const std::vector<std::pair<int, Edge>> &ch, std::vector<double> *alpha_out = nullptr)
    {
        ++lps;
        std::vector<std::vector<double>> E;
        std::vector<double> r;
        for (auto &ce : ch) {
            const Support &s = S[ce.first];
            std::vector<double> row(n);
            for (int j = 0; j < n; ++j) row[j] = s.a[ce.second.p][j] - s.a[ce.second.q][j];
            E.push_back(row);
            r.push_back(s.w[ce.second.q] - s.w[ce.second.p]);
        }
        std::vector<double> a0, N;
        int d = 0;
        if (!nullspace(n, E, r, a0, N, d)) return -INFINITY;
        // inequalities: for every involved support k and b not in the edge: <b - a_p, alpha> >= w_p - w_b + t
        std::vector<double> M, bb;
        int m = 0;
        double scale = 1.0;
        for (auto &ce : ch) {
            const Support &s = S[ce.first];
            const int P = ce.second.p;
            for (int i = 0; i < (int)s.a.size(); ++i) {
                if (i == ce.second.p || i == ce.second.q) continue;
                std::vector<double> g(n);
                for (int j = 0; j < n; ++j) g[j] = s.a[i][j] - s.a[P][j];
                double h = s.w[P] - s.w[i];
                double ga0 = 0.0;
                for (int j = 0; j < n; ++j) ga0 += g[j] * a0[j];
                // -(gN) beta + t <= g a0 - h
                for (int f = 0; f < d; ++f) {
                    double v = 0.0;
                    for (int j = 0; j < n; ++j) v += g[j] * N[(size_t)j * d + f];
                    M.push_back(-v);
                }
                M.push_back(1.0);
                bb.push_back(ga0 - h);
                scale = std::max(scale, std::fabs(ga0 - h));
                ++m;
            }
        }
        if (m == 0) return 1.0;
        if (d == 0) {
            double t = INFINITY;
            for (int i = 0; i < m; ++i) t = std::min(t, bb[i]);
            if (alpha_out) *alpha_out = a0;
            return std::min(t, 1.0);
        }
        // cap row t <= 1
        for (int f = 0; f < d; ++f) M.push_back(0.0);
        M.push_back(1.0);
        bb.push_back(1.0);
        ++m;
        return lp_max_last(M, bb, m, d + 1);
    }

    void lower_edges()
    {
        edges.assign(n, {});
        for (int k = 0; k < n; ++k) {
            const int m = (int)S[k].a.size();
            for (int p = 0; p < m; ++p)
                for (int q = p + 1; q < m; ++q) {
                    std::vector<std::pair<int, Edge>> ch{{k, Edge{p, q}}};
                    if (margin(ch) > 1e-9) edges[k].push_back(Edge{p, q});
                }
        }
    }
};

} // namespace

extern "C" int64_t mc_cells(int n, const int64_t *off, const int32_t *exps, const double *lift, int64_t max_cells,
                            int32_t *pairs_out, double *alpha_out, double *gap_out, int64_t *stats)
{
    Solver sv;
    sv.n = n;
    sv.S.resize(n);
    for (int k = 0; k < n; ++k) {
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            std::vector<double> a(n);
            for (int j = 0; j < n; ++j) a[j] = exps[i * n + j];
            sv.S[k].a.push_back(a);
            sv.S[k].w.push_back(lift[i]);
            sv.S[k].gid.push_back((int)i);
        }
    }
    sv.lower_edges();
    // pairwise compatibility as bitsets: comp[x][y][i] = edges of y compatible with edge i of x
    std::vector<int> nw(n);
    for (int y = 0; y < n; ++y) nw[y] = ((int)sv.edges[y].size() + 63) / 64;
    std::vector<std::vector<std::vector<std::vector<uint64_t>>>> comp(n, std::vector<std::vector<std::vector<uint64_t>>>(n));
    for (int x = 0; x < n; ++x)
        for (int y = 0; y < n; ++y) {
            if (x == y) continue;
            comp[x][y].assign(sv.edges[x].size(), std::vector<uint64_t>(nw[y], 0));
        }
    for (int x = 0; x < n; ++x)
        for (int y = x + 1; y < n; ++y)
            for (size_t i = 0; i < sv.edges[x].size(); ++i)
                for (size_t j = 0; j < sv.edges[y].size(); ++j) {
                    std::vector<std::pair<int, Edge>> ch{{x, sv.edges[x][i]}, {y, sv.edges[y][j]}};
                    if (sv.margin(ch) > 1e-9) {
                        comp[x][y][i][j / 64] |= 1ull << (j % 64);
                        comp[y][x][j][i / 64] |= 1ull << (i % 64);
                    }
                }
    int64_t ncell = 0;
    bool overflow = false;
    std::vector<std::pair<int, Edge>> chosen;
    std::vector<char> used(n, 0);
    std::vector<double> alpha;
    auto popcnt = [](const std::vector<uint64_t> &b) {
        int c = 0;
        for (uint64_t w : b) c += __builtin_popcountll(w);
        return c;
    };
    // cand[y]: edges of support y compatible (pairwise) with every chosen edge
    auto dfs = [&](auto &&self, std::vector<std::vector<uint64_t>> &cand) -> void {
        if (overflow) return;
        const int level = (int)chosen.size();
        if (level == n) {
            double t = sv.margin(chosen, &alpha);
            if (!(t > 1e-9)) return;
            if (ncell >= max_cells) { overflow = true; return; }
            for (auto &ce : chosen) {
                const int k = ce.first;
                pairs_out[(ncell * n + k) * 2 + 0] = sv.S[k].gid[ce.second.p];
                pairs_out[(ncell * n + k) * 2 + 1] = sv.S[k].gid[ce.second.q];
            }
            for (int j = 0; j < n; ++j) alpha_out[ncell * n + j] = alpha[j];
            double gap = INFINITY;
            for (auto &ce : chosen) {
                const Support &s = sv.S[ce.first];
                const int P = ce.second.p;
                double beta = s.w[P];
                for (int j = 0; j < n; ++j) beta += s.a[P][j] * alpha[j];
                for (int i = 0; i < (int)s.a.size(); ++i) {
                    if (i == ce.second.p || i == ce.second.q) continue;
                    double v = s.w[i] - beta;
                    for (int j = 0; j < n; ++j) v += s.a[i][j] * alpha[j];
                    gap = std::min(gap, v);
                }
            }
            gap_out[ncell] = gap;
            ++ncell;
            return;
        }
        // dynamic ordering: the unused support with the fewest candidates (forward checking)
        int k = -1, best = 1 << 30;
        for (int y = 0; y < n; ++y) {
            if (used[y]) continue;
            int c = popcnt(cand[y]);
            if (c == 0) return;
            if (c < best) { best = c; k = y; }
        }
        used[k] = 1;
        for (int e = 0; e < (int)sv.edges[k].size(); ++e) {
            if (!((cand[k][e / 64] >> (e % 64)) & 1)) continue;
            chosen.push_back({k, sv.edges[k][e]});
            ++sv.nodes;
            if (level + 1 == n || level < 1 || sv.margin(chosen) > 1e-9) {
                std::vector<std::vector<uint64_t>> next(cand);
                bool dead = false;
                for (int y = 0; y < n && !dead; ++y) {
                    if (used[y]) continue;
                    int c = 0;
                    for (int w = 0; w < nw[y]; ++w) {
                        next[y][w] &= comp[k][y][e][w];
                        c += __builtin_popcountll(next[y][w]);
                    }
                    dead = (c == 0);
                }
                if (!dead) self(self, next);
            }
            chosen.pop_back();
        }
        used[k] = 0;
    };
    std::vector<std::vector<uint64_t>> cand0(n);
    for (int y = 0; y < n; ++y) {
        cand0[y].assign(nw[y], 0);
        for (int e = 0; e < (int)sv.edges[y].size(); ++e) cand0[y][e / 64] |= 1ull << (e % 64);
    }
    dfs(dfs, cand0);
    if (stats) {
        stats[0] = sv.lps;
        stats[1] = sv.nodes;
        int64_t ne = 0;
        for (auto &e : sv.edges) ne += (int64_t)e.size();
        stats[2] = ne;
    }
    return overflow ? -1 : ncell;
}
