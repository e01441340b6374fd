// (f1) Locality reordering (§4.4: "rearranging nodes with
// similar neighbors ... to be positioned closer"; Rabbit Reordering is the
// paper's default step and is not reimplemented — SPEC S:403 substitutes a
// BFS family).  Host code: the ordering is per-graph preprocessing, amortised
// over every layer and epoch.
//
//   strategy 0  identity
//   strategy 1  BFS (Cuthill-McKee): components in descending size, each
//               numbered breadth-first from a pseudo-peripheral node (two
//               George-Liu sweeps), neighbours visited in ascending degree
//   strategy 2  degree: nodes by descending degree (stable), which packs the
//               hub rows of B that most nonzeros gather together
//
// perm[old] = new.  The graph is treated as undirected (A + A^T pattern).
#include "guard.h"
#include <algorithm>
#include <numeric>
#include <string>
#include <vector>

#include "pspmm.h"

namespace pspmm {
void set_error(const std::string &msg);
}

namespace {

struct Graph {
  int64_t n;
  std::vector<int64_t> ptr;
  std::vector<int32_t> adj;
};

// symmetrised adjacency without self loops
Graph symmetrize(int64_t n, const int32_t *rowptr, const int32_t *colidx) {
  Graph g;
  g.n = n;
  std::vector<int64_t> deg(n + 1, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      const int64_t j = colidx[p];
      if (j == i) continue;
      deg[i]++;
      deg[j]++;
    }
  g.ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) g.ptr[i + 1] = g.ptr[i] + deg[i];
  g.adj.resize(g.ptr[n]);
  std::vector<int64_t> fill(g.ptr.begin(), g.ptr.end() - 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      const int64_t j = colidx[p];
      if (j == i) continue;
      g.adj[fill[i]++] = (int32_t)j;
      g.adj[fill[j]++] = (int32_t)i;
    }
  // sort + dedup each list (A and A^T may both hold an edge)
  std::vector<int64_t> nptr(n + 1, 0);
  int64_t w = 0;
  for (int64_t i = 0; i < n; ++i) {
    auto b = g.adj.begin() + g.ptr[i], e = g.adj.begin() + g.ptr[i + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    nptr[i] = w;
    for (auto it = b; it != u; ++it) g.adj[w++] = *it;
  }
  nptr[n] = w;
  g.adj.resize(w);
  g.ptr.swap(nptr);
  return g;
}

// BFS from s over unvisited-in-`mark` nodes; returns the visit order (levels)
void bfs(const Graph &g, int32_t s, std::vector<int32_t> &stamp, int32_t tag,
         std::vector<int32_t> &order, std::vector<int32_t> *level, bool by_degree) {
  order.clear();
  order.push_back(s);
  stamp[s] = tag;
  if (level) (*level)[s] = 0;
  std::vector<int32_t> nb;
  for (size_t h = 0; h < order.size(); ++h) {
    const int32_t v = order[h];
    nb.clear();
    for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
      const int32_t u = g.adj[p];
      if (stamp[u] != tag) {
        stamp[u] = tag;
        nb.push_back(u);
      }
    }
    if (by_degree)
      std::stable_sort(nb.begin(), nb.end(), [&](int32_t a, int32_t b) {
        return g.ptr[a + 1] - g.ptr[a] < g.ptr[b + 1] - g.ptr[b];
      });
    for (int32_t u : nb) {
      if (level) (*level)[u] = (*level)[v] + 1;
      order.push_back(u);
    }
  }
}

}  // namespace

extern "C" pspmm_status pspmm_reorder(int64_t n, const int32_t *h_rowptr, const int32_t *h_colidx,
                                      int32_t strategy, int32_t *h_perm) {
  return pspmm::guarded("reorder", [&]() -> pspmm_status {
    if (n < 1 || !h_rowptr || !h_perm || (h_rowptr[n] > 0 && !h_colidx)) {
      pspmm::set_error("reorder: bad arguments");
      return PSPMM_ERR_INVALID_ARG;
    }
    if (strategy == 0) {
      for (int64_t i = 0; i < n; ++i) h_perm[i] = (int32_t)i;
      return PSPMM_OK;
    }
    Graph g = symmetrize(n, h_rowptr, h_colidx);
    auto degree = [&](int64_t v) { return g.ptr[v + 1] - g.ptr[v]; };
    if (strategy == 2) {
      std::vector<int32_t> idx(n);
      std::iota(idx.begin(), idx.end(), 0);
      std::stable_sort(idx.begin(), idx.end(),
                       [&](int32_t a, int32_t b) { return degree(a) > degree(b); });
      for (int64_t k = 0; k < n; ++k) h_perm[idx[k]] = (int32_t)k;
      return PSPMM_OK;
    }
    if (strategy != 1) {
      pspmm::set_error("reorder: strategy must be 0 (identity), 1 (BFS) or 2 (degree)");
      return PSPMM_ERR_CONFIG;
    }
    // components (in node order), then numbered in descending size
    std::vector<int32_t> stamp(n, -1), order, comp_of(n, -1);
    std::vector<std::pair<int64_t, int32_t>> comps;  // (size, representative)
    int32_t tag = 0;
    for (int64_t v = 0; v < n; ++v) {
      if (stamp[v] >= 0) continue;
      bfs(g, (int32_t)v, stamp, tag, order, nullptr, false);
      // lowest-degree node of the component starts the peripheral search
      int32_t best = order[0];
      for (int32_t u : order)
        if (degree(u) < degree(best)) best = u;
      comps.push_back({(int64_t)order.size(), best});
      ++tag;
    }
    std::stable_sort(comps.begin(), comps.end(),
                     [](const auto &a, const auto &b) { return a.first > b.first; });
    std::vector<int32_t> level(n, 0);
    std::vector<int32_t> stamp2(n, -1);
    int64_t next = 0;
    int32_t tag2 = 0;
    for (const auto &c : comps) {
      // George-Liu: two sweeps toward a pseudo-peripheral node
      int32_t s = c.second;
      for (int sweep = 0; sweep < 2; ++sweep) {
        bfs(g, s, stamp2, tag2++, order, &level, false);
        const int32_t far_level = level[order.back()];
        int32_t cand = order.back();
        for (int32_t u : order)
          if (level[u] == far_level && degree(u) < degree(cand)) cand = u;
        s = cand;
      }
      bfs(g, s, stamp2, tag2++, order, nullptr, true);
      for (int32_t u : order) h_perm[u] = (int32_t)(next++);
    }
    return PSPMM_OK;
  });
}
