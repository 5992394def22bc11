// Lexicographically smallest minimum-cost assignment (host, O(n^3)).
//
// Replaces the reference's `hungarian` (permutation.py:199-235): scipy's linear_sum_assignment
// for the optimum, then rows fixed in order, each to the smallest column j for which
//   prefix + C[i][j] + (min-cost completion of rows i+1.. without column j) <= opt + tol,
//   tol = 1e-9 * max(1, sum |C|).
// The reference solves one LSA per (row, candidate) -- O(n^2) LSAs.  Here one optimal matching
// and its dual potentials are carried from row to row: with reduced costs r(a,b) = C[a][b] -
// u[a] - v[b] (>= 0, 0 on matched edges), the cheapest matching that forces (i, j) costs
//   OPT_i + r(i, j) + dist(j)
// where dist(b) is the shortest alternating path from column b back to row i's current column
// (one dense Dijkstra per row over the reversed column graph).  Fixing (i, j) augments along
// that path; u' = u + dist(match), v' = v - dist keeps the duals feasible and tight for the
// remaining rows (standard successive-shortest-path argument).  Same decisions as the
// reference unless a candidate lands within rounding distance of the tolerance boundary.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <limits>
#include <vector>

#include "common.cuh"

namespace {

// numpy's pairwise summation over a contiguous double array (pairwise_sum_DOUBLE)
double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    const int64_t stop = n - (n % 8);
    for (; i < stop; i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t h = n / 2;
  h -= h % 8;
  return np_pairwise(a, h) + np_pairwise(a + h, n - h);
}

// Minimum-cost perfect matching (shortest augmenting paths, Jonker-Volgenant style) with dual
// potentials.  row_of[col], col_of[row]; u (rows), v (cols) feasible: C - u - v >= 0, tight on
// the matching.
void solve_lsa(const double* C, int n, std::vector<int>& col_of, std::vector<int>& row_of,
               std::vector<double>& u, std::vector<double>& v) {
  const double INF = std::numeric_limits<double>::infinity();
  col_of.assign(n, -1);
  row_of.assign(n, -1);
  u.assign(n, 0.0);
  v.assign(n, 0.0);
  std::vector<double> dist(n);
  std::vector<int> pred(n), done(n);
  std::vector<int> touched;
  for (int s = 0; s < n; ++s) {  // add row s
    std::fill(dist.begin(), dist.end(), INF);
    std::fill(done.begin(), done.end(), 0);
    for (int b = 0; b < n; ++b) {
      dist[b] = C[(int64_t)s * n + b] - u[s] - v[b];
      pred[b] = -1;  // -1: reached directly from row s
    }
    touched.clear();
    int sink = -1;
    double dmin = 0.0;
    while (sink < 0) {
      int bmin = -1;
      double best = INF;
      for (int b = 0; b < n; ++b)
        if (!done[b] && (dist[b] < best || (dist[b] == best && bmin < 0))) {
          best = dist[b];
          bmin = b;
        }
      done[bmin] = 1;
      touched.push_back(bmin);
      dmin = best;
      const int r = row_of[bmin];
      if (r < 0) {
        sink = bmin;
        break;
      }
      for (int b = 0; b < n; ++b) {
        if (done[b]) continue;
        const double nd = dmin + (C[(int64_t)r * n + b] - u[r] - v[b]);
        if (nd < dist[b]) {
          dist[b] = nd;
          pred[b] = bmin;
        }
      }
    }
    // potentials (only scanned columns move)
    u[s] += dmin;
    for (int b : touched) {
      if (b == sink) continue;
      const int r = row_of[b];
      const double delta = dmin - dist[b];
      v[b] -= delta;
      u[r] += delta;
    }
    // augment
    int b = sink;
    while (true) {
      const int pb = pred[b];
      const int r = pb < 0 ? s : row_of[pb];
      row_of[b] = r;
      col_of[r] = b;
      if (pb < 0) break;
      b = pb;
    }
  }
}

}  // namespace

extern "C" int hinm_lex_assignment(const double* C, int n, int64_t* assignment) {
  if (n < 0 || (n > 0 && (!C || !assignment))) return HINM_ERR_VALUE;
  if (n == 0) return HINM_OK;
  for (int64_t i = 0; i < (int64_t)n * n; ++i)
    if (!isfinite(C[i])) return HINM_ERR_VALUE;
  std::vector<int> col_of, row_of;
  std::vector<double> u, v;
  solve_lsa(C, n, col_of, row_of, u, v);
  // opt exactly as the reference forms it: sum of C[rows, cols] (rows ascending), pairwise
  std::vector<double> tmp(n);
  for (int r = 0; r < n; ++r) tmp[r] = C[(int64_t)r * n + col_of[r]];
  const double opt = np_pairwise(tmp.data(), n);
  std::vector<double> absC((size_t)n * n);
  for (int64_t i = 0; i < (int64_t)n * n; ++i) absC[i] = fabs(C[i]);
  const double tol = 1e-9 * std::max(1.0, np_pairwise(absC.data(), (int64_t)n * n));

  // C transposed: the per-row Dijkstra reads column bmin of C for every unfixed row
  std::vector<double> CT((size_t)n * n);
  for (int r = 0; r < n; ++r)
    for (int b = 0; b < n; ++b) CT[(size_t)b * n + r] = C[(size_t)r * n + b];
  std::vector<char> col_alive(n, 1);
  std::vector<int> alive(n), open;
  for (int b = 0; b < n; ++b) alive[b] = b;
  std::vector<double> dist(n);
  std::vector<int> next(n), done(n);
  double prefix = 0.0;
  const double INF = std::numeric_limits<double>::infinity();
  for (int i = 0; i < n; ++i) {
    // OPT of the remaining problem (rows i.., alive columns) under the carried matching
    double opt_i = 0.0;
    for (int r = i; r < n; ++r) opt_i += C[(int64_t)r * n + col_of[r]];
    const int ci = col_of[i];
    // reverse Dijkstra from ci: dist[b] = cheapest way to free ci starting by vacating b
    // (row_of[b] moves to b', ..., until some row moves into ci); next[b] = that first b'
    for (int b : alive) {
      dist[b] = INF;
      done[b] = 0;
      next[b] = -1;
    }
    dist[ci] = 0.0;
    // open = alive columns not yet finalised (compacted as they are finalised)
    open.assign(alive.begin(), alive.end());
    while (!open.empty()) {
      int at = -1;
      double best = INF;
      for (int q = 0; q < (int)open.size(); ++q)
        if (dist[open[q]] < best) {
          best = dist[open[q]];
          at = q;
        }
      if (at < 0) break;
      const int bmin = open[at];
      open[at] = open.back();
      open.pop_back();
      done[bmin] = 1;
      // a row r (unfixed, r != i) may vacate its column b = col_of[r] by moving into bmin;
      // rows are walked in order so column bmin of C is read contiguously from CT
      const double* ct = CT.data() + (size_t)bmin * n;
      const double vb = v[bmin];
      for (int r = i + 1; r < n; ++r) {
        const int b = col_of[r];
        if (done[b]) continue;
        const double nd = best + (ct[r] - u[r] - vb);
        if (nd < dist[b]) {
          dist[b] = nd;
          next[b] = bmin;
        }
      }
    }
    // smallest column whose forced optimum stays within the reference's tolerance
    int jsel = -1;
    for (int j = 0; j < n; ++j) {
      if (!col_alive[j]) continue;
      double forced;
      if (j == ci) {
        forced = opt_i;
      } else {
        const double red = C[(int64_t)i * n + j] - u[i] - v[j];
        forced = opt_i + (red + dist[j]);
      }
      if (prefix + forced <= opt + tol) {
        jsel = j;
        break;
      }
    }
    if (jsel < 0) jsel = ci;  // unreachable in exact arithmetic (ci itself is optimal)
    // augment: row i takes jsel; the row holding jsel follows the path to ci
    if (jsel != ci) {
      // duals for the remaining rows: u' = u + dist(match), v' = v - dist
      for (int r = i + 1; r < n; ++r) u[r] += dist[col_of[r]];
      for (int b = 0; b < n; ++b)
        if (col_alive[b] && dist[b] < INF) v[b] -= dist[b];
      int b = jsel;
      int r = row_of[b];
      while (b != ci) {
        const int nb = next[b];
        const int rn = row_of[nb];  // row currently at nb (row i when nb == ci)
        row_of[nb] = r;
        col_of[r] = nb;
        b = nb;
        r = rn;
      }
      row_of[jsel] = i;
      col_of[i] = jsel;
    }
    assignment[i] = jsel;
    prefix += C[(int64_t)i * n + jsel];
    col_alive[jsel] = 0;
    alive.erase(std::find(alive.begin(), alive.end(), jsel));
  }
  return HINM_OK;
}
