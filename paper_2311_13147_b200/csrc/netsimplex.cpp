// NEXT-4: the small LOT of Theorem 1 (eq. small_problem_CLOT; Alg. 1 line 2,
// P:332-347) by the primal network simplex method the paper names, host C++.
//
// The transportation problem min <G, S> s.t. S 1 = alpha, S^T 1 = beta, S >= 0 is a min-cost flow on the
// complete bipartite graph: m source nodes (supply alpha_i), m sink nodes (demand beta_j), arcs i -> m+j
// of cost G_ij and unbounded capacity. Design (SPEC's ledger):
//   * masses are scaled to 64-bit integers (total 2^50) so that every flow update is exact integer
//     arithmetic; the flow is rescaled at the end;
//   * the initial basis is the strongly feasible artificial tree (every node hangs from a root node by an
//     artificial arc of cost M carrying its supply / demand), and the leaving arc is chosen by the strongly
//     feasible rule (the last blocking arc when the pivot cycle is traversed in the direction of the
//     entering arc from the apex), so degenerate pivots cannot cycle;
//   * entering arcs by block search (blocks of ~m arcs, the most negative reduced cost of the block; ties to
//     the first in scan order), restarting where the previous search stopped (deterministic);
//   * after each pivot the tree's depth / preorder / potentials are recomputed by one DFS from the root
//     (O(m) per pivot, like the block search).
// Output: the plan S (a vertex: at most 2m - 1 non-zeros), its value, and dual potentials (u, v) with
// u_i + v_j <= G_ij and equality on the support (the optimality certificate, P:365-367 for phi = 0).
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/cyclicot.h"

namespace cot {
void set_error(const std::string& msg);
}

namespace {

struct NetworkSimplex {
  int m, nn, root;                       // nodes: sources [0, m), sinks [m, 2m), root 2m
  const double* G;
  // arcs: real arcs a = i * m + j (i -> m + j); artificial arc of node v: A + v (v -> root for sources,
  // root -> v for sinks)
  int64_t A;
  std::vector<int64_t> flow;             // [A + 2m]
  std::vector<int> parent, depth;        // tree
  std::vector<int64_t> pred;             // arc joining v to parent[v]
  std::vector<double> pi;                // node potentials: reduced cost c_a - pi[tail] + pi[head]
  std::vector<int> order, first_child, next_sib, stack, upath;
  double M;                              // artificial cost
  int64_t search_pos = 0;
  int64_t pivots = 0;

  int tail(int64_t a) const { return a < A ? (int)(a / m) : (int)(a - A) < m ? (int)(a - A) : root; }
  int head(int64_t a) const { return a < A ? m + (int)(a % m) : (int)(a - A) < m ? root : (int)(a - A); }
  double cost(int64_t a) const { return a < A ? G[a] : M; }

  void rebuild() {   // children lists from parent[], then DFS: depth, preorder, potentials
    std::fill(first_child.begin(), first_child.end(), -1);
    for (int v = nn - 1; v >= 0; --v)
      if (v != root) {
        next_sib[v] = first_child[parent[v]];
        first_child[parent[v]] = v;
      }
    order.clear();
    stack.clear();
    stack.push_back(root);
    depth[root] = 0;
    pi[root] = 0.0;
    while (!stack.empty()) {
      const int v = stack.back();
      stack.pop_back();
      order.push_back(v);
      for (int c = first_child[v]; c >= 0; c = next_sib[c]) {
        depth[c] = depth[v] + 1;
        const int64_t a = pred[c];
        // tree arcs have zero reduced cost: c_a - pi[tail] + pi[head] = 0
        if (tail(a) == c) pi[c] = cost(a) + pi[v];      // arc c -> v
        else pi[c] = pi[v] - cost(a);                   // arc v -> c
        stack.push_back(c);
      }
    }
  }

  // block search for an entering real arc with negative reduced cost: the most negative of a block of ~m
  // arcs (first in scan order on ties), scanning cyclically from where the previous search stopped
  int64_t find_entering(double tol) {
    const int64_t block = std::max<int64_t>(m, 64);
    int64_t best = -1;
    double bestrc = -tol;
    int64_t scanned = 0;
    int64_t a = search_pos;
    while (scanned < A) {
      const int64_t end = std::min<int64_t>(scanned + block, A);
      for (; scanned < end; ++scanned) {
        const double rc = G[a] - pi[(size_t)(a / m)] + pi[(size_t)(m + a % m)];
        if (rc < bestrc) {
          bestrc = rc;
          best = a;
        }
        if (++a == A) a = 0;
      }
      if (best >= 0) {
        search_pos = a;
        return best;
      }
    }
    return -1;
  }

  // one pivot on entering arc e = (u -> w)
  void pivot(int64_t e) {
    const int u = tail(e), w = head(e);
    // apex: common ancestor of u and w
    int x = u, y = w;
    while (x != y) {
      if (depth[x] >= depth[y]) x = parent[x];
      else y = parent[y];
    }
    const int apex = x;
    // the cycle, oriented along e: apex -> ... -> u -> w -> ... -> apex. Arcs on the u side are traversed
    // from parent to child (apex down to u); on the w side from child to parent (w up to apex). An arc is
    // forward if its direction agrees with the orientation (flow += delta), backward otherwise (flow -=).
    // Strongly feasible rule: the leaving arc is the LAST blocking (min-flow backward) arc along the
    // orientation starting at the apex.
    int64_t delta = INT64_MAX;
    int leave_node = -1;      // the child endpoint of the leaving tree arc
    bool leave_on_u_side = false;
    // u side in orientation order: apex ... u, i.e. reverse of the climb from u. Collect the climb.
    upath.clear();
    for (int v = u; v != apex; v = parent[v]) upath.push_back(v);
    for (int k = (int)upath.size() - 1; k >= 0; --k) {   // apex -> u order
      const int v = upath[k];
      const int64_t a = pred[v];
      const bool forward = head(a) == v;   // traversed parent -> v
      if (!forward && flow[a] <= delta) {  // '<=' keeps the last blocking arc
        delta = flow[a];
        leave_node = v;
        leave_on_u_side = true;
      }
    }
    for (int v = w; v != apex; v = parent[v]) {   // w -> apex order (after e in the orientation)
      const int64_t a = pred[v];
      const bool forward = tail(a) == v;   // traversed v -> parent
      if (!forward && flow[a] <= delta) {
        delta = flow[a];
        leave_node = v;
        leave_on_u_side = false;
      }
    }
    if (delta == INT64_MAX) {   // cannot happen with finite supplies (unbounded problem)
      delta = 0;
    }
    // flow update along the cycle
    flow[e] += delta;
    for (int v = u; v != apex; v = parent[v]) {
      const int64_t a = pred[v];
      if (head(a) == v) flow[a] += delta; else flow[a] -= delta;
    }
    for (int v = w; v != apex; v = parent[v]) {
      const int64_t a = pred[v];
      if (tail(a) == v) flow[a] += delta; else flow[a] -= delta;
    }
    // tree update: remove pred[leave_node], add e; the subtree that hung below leave_node is re-rooted at
    // the endpoint of e on its side (u if the leaving arc was on the u side, else w)
    int v = leave_on_u_side ? u : w;
    int new_parent = leave_on_u_side ? w : u;
    int64_t new_pred = e;
    // reverse the parent pointers on the path v -> ... -> leave_node
    while (true) {
      const int old_parent = parent[v];
      const int64_t old_pred = pred[v];
      parent[v] = new_parent;
      pred[v] = new_pred;
      if (v == leave_node) break;
      new_parent = v;
      new_pred = old_pred;
      v = old_parent;
    }
    rebuild();
    ++pivots;
  }
};

}  // namespace

extern "C" int clot_small_lot(const double* alpha, const double* beta, const double* G, int64_t m, double* S,
                              double* value, double* u, double* v, int64_t* pivots) {
  if (m < 1 || m > 46340 || !alpha || !beta || !G || !S) {
    cot::set_error("clot_small_lot: need 1 <= m <= 46340 and non-NULL alpha, beta, G, S");
    return COT_E_ARG;
  }
  double sa = 0.0, sb = 0.0, gmax = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    if (!(alpha[i] > 0.0) || !(beta[i] > 0.0) || !std::isfinite(alpha[i]) || !std::isfinite(beta[i])) {
      cot::set_error("clot_small_lot: alpha and beta must be finite and > 0");
      return COT_E_MARGINAL;
    }
    sa += alpha[i];
    sb += beta[i];
  }
  if (std::fabs(sa - sb) > 1e-6 * std::max(sa, sb)) {
    cot::set_error("clot_small_lot: sum(alpha) != sum(beta)");
    return COT_E_MARGINAL;
  }
  for (int64_t k = 0; k < m * m; ++k) {
    if (!std::isfinite(G[k])) {
      cot::set_error("clot_small_lot: non-finite cost");
      return COT_E_NONFINITE;
    }
    gmax = std::max(gmax, std::fabs(G[k]));
  }
  // integer masses: total 2^50, rounding residue on the largest entry
  const double total = 1125899906842624.0;   // 2^50
  auto scale = [&](const double* x, double s, std::vector<int64_t>& out) {
    out.resize((size_t)m);
    int64_t acc = 0;
    int64_t big = 0;
    for (int64_t i = 0; i < m; ++i) {
      out[(size_t)i] = std::max<int64_t>(1, (int64_t)std::llround(x[i] / s * total));
      acc += out[(size_t)i];
      if (out[(size_t)i] > out[(size_t)big]) big = i;
    }
    out[(size_t)big] += (int64_t)total - acc;
  };
  std::vector<int64_t> ai, bi;
  scale(alpha, sa, ai);
  scale(beta, sb, bi);

  NetworkSimplex ns;
  ns.m = (int)m;
  ns.nn = 2 * (int)m + 1;
  ns.root = 2 * (int)m;
  ns.G = G;
  ns.A = m * m;
  ns.M = (gmax + 1.0) * (double)(2 * m + 1);
  ns.flow.assign((size_t)(ns.A + 2 * m), 0);
  ns.parent.assign((size_t)ns.nn, ns.root);
  ns.depth.assign((size_t)ns.nn, 1);
  ns.pred.assign((size_t)ns.nn, -1);
  ns.pi.assign((size_t)ns.nn, 0.0);
  ns.first_child.assign((size_t)ns.nn, -1);
  ns.next_sib.assign((size_t)ns.nn, -1);
  for (int64_t i = 0; i < m; ++i) {   // artificial tree: sources -> root, root -> sinks
    ns.pred[(size_t)i] = ns.A + i;
    ns.flow[(size_t)(ns.A + i)] = ai[(size_t)i];
    ns.pred[(size_t)(m + i)] = ns.A + m + i;
    ns.flow[(size_t)(ns.A + m + i)] = bi[(size_t)i];
  }
  ns.parent[(size_t)ns.root] = -1;
  ns.rebuild();
  const double tol = 1e-11 * std::max(1.0, gmax);   // above the rounding of potentials of size ~M
  const int64_t max_pivots = 200 * m * m + 100000;
  while (true) {
    const int64_t e = ns.find_entering(tol);
    if (e < 0) break;
    ns.pivot(e);
    if (ns.pivots > max_pivots) {
      cot::set_error("clot_small_lot: pivot limit exceeded");
      return COT_E_ARG;
    }
  }
  for (int64_t k = 0; k < 2 * m; ++k)
    if (ns.flow[(size_t)(ns.A + k)] != 0) {
      cot::set_error("clot_small_lot: artificial flow left (infeasible)");
      return COT_E_MARGINAL;
    }
  double val = 0.0;
  for (int64_t a = 0; a < ns.A; ++a) {
    S[a] = (double)ns.flow[(size_t)a] / total * sa;
    val += G[a] * S[a];
  }
  if (value) *value = val;
  // duals: reduced cost G_ij - pi_i + pi_{m+j} >= 0  =>  u_i = pi_i - pi_root, v_j = pi_root - pi_{m+j}
  if (u)
    for (int64_t i = 0; i < m; ++i) u[i] = ns.pi[(size_t)i];
  if (v)
    for (int64_t j = 0; j < m; ++j) v[j] = -ns.pi[(size_t)(m + j)];
  if (pivots) *pivots = ns.pivots;
  return COT_OK;
}

// Theorem 1 with the full-scale factor of P:251: the optimal value of the explicit d x d C-LOT problem is
// n times the small LOT's <G, S*>. The library applies the factor (callers need not know the reduction's scaling).
extern "C" int clot_lot_value(const double* alpha, const double* beta, const double* G, int64_t m, int64_t n,
                              double* S, double* value_full, double* value_small) {
  if (n < 1 || !value_full) {
    cot::set_error("clot_lot_value: need n >= 1 and value_full");
    return COT_E_ARG;
  }
  double small = 0.0;
  const int st = clot_small_lot(alpha, beta, G, m, S, &small, nullptr, nullptr, nullptr);
  if (st != COT_OK) return st;
  *value_full = (double)n * small;
  if (value_small) *value_small = small;
  return COT_OK;
}
