// Host symbolic analysis shared by every shift (one
// fill-reducing ordering per sparsity pattern, reused across shifts).
//
//  1. Geometric nested dissection on the DoF coordinates.  A region is split
//     by a grid line x_axis == c (axis = longer bounding-box side) chosen as
//     close to the median as possible among lines that really separate the
//     graph (no edge between x < c and x > c).  For P1 right-triangle meshes
//     every grid line separates; for P2 only the coarse lines do, and the
//     check finds them.  If no line separates, the vertex separator of the
//     median edge cut is used.  Regions of <= leaf_size DoFs become leaves.
//  2. Postorder numbering: left subtree, right subtree, separator.
//  3. Fronts = tree nodes; boundary rows B_s = (adj(pivots) U children's B)
//     restricted to indices after the front's last pivot (all in ancestors).
//  4. Extend-add maps (child boundary row -> parent front position), original
//     entry maps (CSR lower entry -> factor block slot), memory offsets.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>
#include <string>

#include "plan.h"

namespace stfem {
namespace {

struct TreeNode {
  std::vector<int32_t> piv;   // old DoF ids
  std::vector<int32_t> kids;  // tree node ids
};

struct ND {
  int32_t n, dim, leaf;
  const int64_t* rp;
  const int32_t* ci;
  const double* xy;
  std::vector<TreeNode> nodes;
  std::vector<int32_t> stamp;
  int32_t cur = 0;

  double coord(int32_t v, int axis) const { return xy[(int64_t)v * dim + axis]; }

  void order_by(std::vector<int32_t>& S, int primary) {
    int secondary = dim == 2 ? 1 - primary : primary;
    std::sort(S.begin(), S.end(), [&](int32_t a, int32_t b) {
      double pa = coord(a, primary), pb = coord(b, primary);
      if (pa != pb) return pa < pb;
      double sa = coord(a, secondary), sb = coord(b, secondary);
      if (sa != sb) return sa < sb;
      return a < b;
    });
  }

  // true iff no edge joins x_axis < c and x_axis > c inside the stamped region
  bool separates(const std::vector<int32_t>& S, int axis, double c) {
    for (int32_t u : S) {
      if (!(coord(u, axis) < c)) continue;
      for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
        int32_t v = ci[k];
        if (stamp[v] == cur && coord(v, axis) > c) return false;
      }
    }
    return true;
  }

  int32_t build(std::vector<int32_t>& S) {
    int32_t id = (int32_t)nodes.size();
    nodes.emplace_back();
    if ((int32_t)S.size() <= leaf) {
      order_by(S, 1 % dim);
      nodes[id].piv = S;
      return id;
    }
    double lo[2] = {1e300, 1e300}, hi[2] = {-1e300, -1e300};
    for (int32_t v : S)
      for (int a = 0; a < dim; ++a) {
        lo[a] = std::min(lo[a], coord(v, a));
        hi[a] = std::max(hi[a], coord(v, a));
      }
    int axis = (dim == 2 && hi[1] - lo[1] > hi[0] - lo[0]) ? 1 : 0;
    std::vector<double> vals(S.size());
    for (size_t i = 0; i < S.size(); ++i) vals[i] = coord(S[i], axis);
    std::vector<double> sorted = vals;
    std::sort(sorted.begin(), sorted.end());
    double med = sorted[sorted.size() / 2];
    std::vector<double> dv = sorted;
    dv.erase(std::unique(dv.begin(), dv.end()), dv.end());
    ++cur;
    for (int32_t v : S) stamp[v] = cur;

    int m0 = (int)(std::lower_bound(dv.begin(), dv.end(), med) - dv.begin());
    double cut = 0;
    bool found = false;
    if (dv.size() >= 3) {
      for (int off = 0; off < 16 && !found; ++off) {
        for (int sgn = 0; sgn < 2 && !found; ++sgn) {
          int idx = sgn ? m0 - off : m0 + off;
          if (off == 0 && sgn) continue;
          if (idx <= 0 || idx >= (int)dv.size() - 1) continue;  // both sides non-empty
          if (separates(S, axis, dv[idx])) {
            cut = dv[idx];
            found = true;
          }
        }
      }
    }
    std::vector<int32_t> L, R, sep;
    if (found) {
      for (int32_t v : S) {
        double x = coord(v, axis);
        (x < cut ? L : (x > cut ? R : sep)).push_back(v);
      }
    } else {
      // vertex separator of the median edge cut: R-nodes adjacent to L
      cut = med;
      if (cut == dv.front() && dv.size() > 1) cut = dv[1];
      for (int32_t v : S) {
        if (coord(v, axis) < cut) {
          L.push_back(v);
          continue;
        }
        bool touches = false;
        for (int64_t k = rp[v]; k < rp[v + 1] && !touches; ++k) {
          int32_t u = ci[k];
          touches = stamp[u] == cur && coord(u, axis) < cut;
        }
        (touches ? sep : R).push_back(v);
      }
      if (sep.empty()) {  // disconnected halves: keep a one-node separator
        if (!R.empty()) {
          sep.push_back(R.back());
          R.pop_back();
        } else {
          sep.push_back(L.back());
          L.pop_back();
        }
      }
    }
    std::vector<int32_t> kids;
    if (!L.empty()) kids.push_back(build(L));
    if (!R.empty()) kids.push_back(build(R));
    order_by(sep, dim == 2 ? 1 - axis : 0);
    nodes[id].piv = std::move(sep);
    nodes[id].kids = std::move(kids);
    return id;
  }
};

}  // namespace

int build_symbolic(Plan& P, int32_t n, const int64_t* rowptr, const int32_t* colind,
                   const double* coords, int32_t dim, int32_t leaf_size) {
  if (n <= 0) return fail(STFEM_ERR_DIM, "plan: n must be positive (no interior DoFs)");
  if (dim != 1 && dim != 2) return fail(STFEM_ERR_ARG, "plan: dim must be 1 or 2");
  if (leaf_size < 1) leaf_size = 32;
  for (int32_t r = 0; r < n; ++r)
    if (rowptr[r + 1] < rowptr[r]) return fail(STFEM_ERR_ARG, "plan: rowptr not monotone");
  const int64_t nnz = rowptr[n];
  for (int64_t k = 0; k < nnz; ++k)
    if (colind[k] < 0 || colind[k] >= n) return fail(STFEM_ERR_ARG, "plan: column index out of range");

  P.n = n;
  P.nnz_pattern = nnz;
  ND nd{n, dim, leaf_size, rowptr, colind, coords, {}, std::vector<int32_t>(n, 0), 0};
  std::vector<int32_t> all(n);
  std::iota(all.begin(), all.end(), 0);
  int32_t root = nd.build(all);

  // ---- postorder numbering -> fronts ----
  P.perm.assign(n, -1);
  P.iperm.assign(n, -1);
  P.fronts.clear();
  std::vector<int32_t> node2front(nd.nodes.size(), -1);
  std::vector<int32_t> node_depth(nd.nodes.size(), 0);
  int32_t next = 0;
  // iterative postorder
  std::vector<std::pair<int32_t, int32_t>> st{{root, 0}};
  while (!st.empty()) {
    auto& [id, k] = st.back();
    if (k < (int32_t)nd.nodes[id].kids.size()) {
      int32_t kid = nd.nodes[id].kids[k++];
      node_depth[kid] = node_depth[id] + 1;
      st.push_back({kid, 0});
      continue;
    }
    FrontDev f{};
    f.pbeg = next;
    f.p = (int32_t)nd.nodes[id].piv.size();
    f.depth = node_depth[id];
    for (int32_t v : nd.nodes[id].piv) {
      P.perm[next] = v;
      P.iperm[v] = next;
      ++next;
    }
    node2front[id] = (int32_t)P.fronts.size();
    P.fronts.push_back(f);
    st.pop_back();
  }
  if (next != n) return fail(STFEM_ERR_INTERNAL, "plan: nested dissection lost DoFs");
  const int32_t nf = (int32_t)P.fronts.size();
  std::vector<std::vector<int32_t>> kids(nf);
  for (size_t id = 0; id < nd.nodes.size(); ++id) {
    int32_t f = node2front[id];
    P.fronts[f].parent = -1;
    for (int32_t kid : nd.nodes[id].kids) kids[f].push_back(node2front[kid]);
  }
  for (int32_t f = 0; f < nf; ++f)
    for (int32_t c : kids[f]) P.fronts[c].parent = f;

  // ---- boundary sets, extend-add maps ----
  std::vector<std::vector<int32_t>> B(nf);
  std::vector<int32_t> mark(n, -1), pos(n, -1);
  P.child_ids.clear();
  P.relpos.assign(0, 0);
  P.bidx.clear();
  std::vector<int32_t> owner(n);
  for (int32_t f = 0; f < nf; ++f) {
    FrontDev& F = P.fronts[f];
    const int32_t pend = F.pbeg + F.p;
    for (int32_t i = F.pbeg; i < pend; ++i) owner[i] = f;
    std::vector<int32_t> b;
    for (int32_t i = F.pbeg; i < pend; ++i) {
      int32_t v = P.perm[i];
      for (int64_t k = rowptr[v]; k < rowptr[v + 1]; ++k) {
        int32_t w = P.iperm[colind[k]];
        if (w >= pend && mark[w] != f) {
          mark[w] = f;
          b.push_back(w);
        }
      }
    }
    for (int32_t c : kids[f])
      for (int32_t w : B[c]) {
        if (w >= pend && mark[w] != f) {
          mark[w] = f;
          b.push_back(w);
        } else if (w < F.pbeg) {
          return fail(STFEM_ERR_INTERNAL, "plan: child boundary row outside the parent front "
                                          "(nested dissection separator leak)");
        }
      }
    std::sort(b.begin(), b.end());
    B[f] = std::move(b);
    F.n = F.p + (int32_t)B[f].size();
    // positions in this front
    for (int32_t i = 0; i < F.p; ++i) pos[F.pbeg + i] = i;
    for (size_t k = 0; k < B[f].size(); ++k) pos[B[f][k]] = F.p + (int32_t)k;
    F.child_beg = (int32_t)P.child_ids.size();
    F.nchild = (int32_t)kids[f].size();
    if (kids[f].size() > 2) return fail(STFEM_ERR_INTERNAL, "plan: front with more than two children");
    F.inv_beg = (int32_t)P.inv.size();
    for (size_t s = 0; s < kids[f].size(); ++s) {
      const int32_t c = kids[f][s];
      P.child_ids.push_back(c);
      FrontDev& Cf = P.fronts[c];
      Cf.relpos_beg = (int32_t)P.relpos.size();
      for (int32_t w : B[c]) P.relpos.push_back(pos[w]);
      // inverse map (parent row -> child boundary row) for the gather assembly
      const size_t base = P.inv.size();
      P.inv.resize(base + F.n, -1);
      for (size_t k = 0; k < B[c].size(); ++k) P.inv[base + pos[B[c][k]]] = (int32_t)k;
    }
    F.bidx_beg = (int32_t)P.bidx.size();
    P.bidx.insert(P.bidx.end(), B[f].begin(), B[f].end());
  }

  // ---- original entries: lower triangle (new numbering) -> factor slot ----
  std::vector<int32_t> cnt(nf + 1, 0);
  std::vector<int32_t> e_front, e_src, e_dst;
  e_front.reserve(nnz / 2 + n);
  P.diag_src.assign(n, -1);   // CSR slot of every diagonal entry (pivot-collapse scale, factor_solve)
  for (int32_t r = 0; r < n; ++r) {
    int32_t i = P.iperm[r];
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
      if (colind[k] == r) P.diag_src[r] = (int32_t)k;
      int32_t j = P.iperm[colind[k]];
      if (i < j) continue;
      int32_t f = owner[j];
      const FrontDev& F = P.fronts[f];
      int32_t pi;
      if (i < F.pbeg + F.p) {
        pi = i - F.pbeg;
      } else {
        auto it = std::lower_bound(B[f].begin(), B[f].end(), i);
        if (it == B[f].end() || *it != i)
          return fail(STFEM_ERR_INTERNAL, "plan: entry row missing from its front");
        pi = F.p + (int32_t)(it - B[f].begin());
      }
      e_front.push_back(f);
      e_src.push_back((int32_t)k);
      e_dst.push_back((j - F.pbeg) * F.n + pi);
      cnt[f + 1]++;
    }
  }
  for (int32_t f = 0; f < nf; ++f) cnt[f + 1] += cnt[f];
  P.ent_colptr.clear();
  P.ent_src.assign(e_src.size(), 0);
  P.ent_dst.assign(e_src.size(), 0);
  {
    std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
    for (size_t e = 0; e < e_src.size(); ++e) {
      int32_t q = fill[e_front[e]]++;
      P.ent_src[q] = e_src[e];
      P.ent_dst[q] = e_dst[e];
    }
  }
  for (int32_t f = 0; f < nf; ++f) {
    P.fronts[f].ent_beg = cnt[f];
    P.fronts[f].ent_cnt = cnt[f + 1] - cnt[f];
    // column-major order within the front: a column block's entries are one
    // contiguous range (the large-front assembly binary-searches it)
    std::vector<std::pair<int32_t, int32_t>> ed(P.fronts[f].ent_cnt);
    for (int32_t q = 0; q < P.fronts[f].ent_cnt; ++q)
      ed[q] = {P.ent_dst[cnt[f] + q], P.ent_src[cnt[f] + q]};
    std::sort(ed.begin(), ed.end());
    for (int32_t q = 0; q < P.fronts[f].ent_cnt; ++q) {
      P.ent_dst[cnt[f] + q] = ed[q].first;
      P.ent_src[cnt[f] + q] = ed[q].second;
    }
    // column pointers: entries of pivot column c are [colptr[c], colptr[c+1])
    FrontDev& F = P.fronts[f];
    F.colptr_beg = (int32_t)P.ent_colptr.size();
    int32_t q = 0;
    for (int32_t c = 0; c <= F.p; ++c) {
      while (q < F.ent_cnt && ed[q].first < c * F.n) ++q;
      P.ent_colptr.push_back(q);
    }
  }

  // ---- levels, offsets, statistics ----
  P.depth = 0;
  for (auto& F : P.fronts) P.depth = std::max(P.depth, F.depth);
  P.levels.assign(P.depth + 1, {});
  for (int32_t f = 0; f < nf; ++f) P.levels[P.fronts[f].depth].push_back(f);
  P.factor_stride = 0;
  P.nnz_factor = 0;
  P.flops = 0;
  P.max_front = P.max_pivots = 0;
  for (auto& F : P.fronts) {
    int64_t b = F.n - F.p;
    P.nnz_factor += (int64_t)F.p * (F.p + 1) / 2 + b * F.p;
    for (int32_t j = 0; j < F.p; ++j) {
      double c = (double)(F.n - 1 - j);
      P.flops += 4.0 * c * c;
    }
    P.max_front = std::max(P.max_front, F.n);
    P.max_pivots = std::max(P.max_pivots, F.p);
  }
  P.levels_all = P.levels;
  P.subs.clear();
  P.sub_levels.assign(P.depth + 1, {});
  assign_factor_offsets(P, std::vector<char>(nf, 0));
  P.upool_stride[0] = P.upool_stride[1] = 0;
  P.rpool_stride[0] = P.rpool_stride[1] = 0;
  for (int32_t d = 0; d <= P.depth; ++d) {
    int64_t u = 0, r = 0;
    for (int32_t f : P.levels[d]) {
      FrontDev& F = P.fronts[f];
      int64_t b = F.n - F.p;
      F.uofs = u;
      F.rofs = r;
      u += (int64_t)ldu((int)b) * b;
      r += b;
    }
    P.upool_stride[d & 1] = std::max(P.upool_stride[d & 1], u);
    P.rpool_stride[d & 1] = std::max(P.rpool_stride[d & 1], r);
  }
  P.uofs0.resize(nf);
  for (int32_t f = 0; f < nf; ++f) P.uofs0[f] = P.fronts[f].uofs;
  return STFEM_OK;
}

void assign_factor_offsets(Plan& P, const std::vector<char>& skip) {
  P.factor_stride = 0;
  for (size_t f = 0; f < P.fronts.size(); ++f) {
    FrontDev& F = P.fronts[f];
    F.fofs = P.factor_stride;
    if (!skip[f]) P.factor_stride += (int64_t)F.n * F.p;
  }
}

}  // namespace stfem
