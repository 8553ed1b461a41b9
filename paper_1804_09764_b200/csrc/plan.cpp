// plan.cpp -- the template partitioner (host, once per template).
//
// pick the root rho(T), cut an edge
// (rho(T), u); T' keeps the root, T'' is rooted at u; recurse until single
// vertices.  Here T is split at its root by cutting the edge to the LAST
// child: sub-template (x, j) = template vertex x with its first j children's
// full subtrees; (x, j) = active (x, j-1) + passive (c_j, all children).
// Isomorphic sub-templates (same AHU canonical code) share one table
// (SPEC "dedup").  The over-count factor d of Eq. 1
// is NOT applied: the DP counts maps and the estimator
// divides by |Aut(T)| once (reading C-1).
#include <algorithm>
#include <functional>
#include <map>

#include "common.h"

namespace cc {

namespace {

struct Tree {
  int k = 0, root = -1;
  std::vector<int> parent;
  std::vector<std::vector<int>> child;  // increasing index order
  std::vector<int> size;
};

Tree load_tree(int k, const int32_t *parent) {
  if (k < 1 || k > kMaxK) throw Error(CC_ERR_TEMPLATE, "template size k must be in [1, 16]");
  if (!parent) throw Error(CC_ERR_ARG, "parent array is NULL");
  Tree T;
  T.k = k;
  T.parent.assign(parent, parent + k);
  T.child.assign(k, {});
  for (int i = 0; i < k; ++i) {
    if (parent[i] == -1) {
      if (T.root >= 0) throw Error(CC_ERR_TEMPLATE, "parent array has more than one -1 (root)");
      T.root = i;
    } else if (parent[i] < 0 || parent[i] >= k || parent[i] == i) {
      throw Error(CC_ERR_TEMPLATE, "parent[" + std::to_string(i) + "] out of range");
    } else {
      T.child[parent[i]].push_back(i);
    }
  }
  if (T.root < 0) throw Error(CC_ERR_TEMPLATE, "parent array has no root (-1)");
  // connected: every vertex reaches the root without a cycle
  for (int i = 0; i < k; ++i) {
    int x = i, steps = 0;
    while (x != T.root) {
      x = T.parent[x];
      if (++steps > k) throw Error(CC_ERR_TEMPLATE, "parent pointers contain a cycle");
    }
  }
  T.size.assign(k, 0);
  std::function<int(int)> sz = [&](int x) {
    int s = 1;
    for (int c : T.child[x]) s += sz(c);
    return T.size[x] = s;
  };
  sz(T.root);
  return T;
}

// AHU canonical code of the subtree of x in the tree rooted at `root`,
// over the undirected adjacency (used for the root orbit).
std::string rooted_code(const std::vector<std::vector<int>> &adj, int x, int from) {
  std::vector<std::string> cs;
  for (int y : adj[x])
    if (y != from) cs.push_back(rooted_code(adj, y, x));
  std::sort(cs.begin(), cs.end());
  std::string s = "(";
  for (auto &c : cs) s += c;
  return s + ")";
}

int64_t factorial(int m) {
  int64_t f = 1;
  for (int i = 2; i <= m; ++i) f *= i;
  return f;
}

}  // namespace

// The same tree rooted at w; children ordered by `order` (0 = vertex index,
// 1 = subtree size ascending, 2 = subtree size descending; ties by index).
Tree reroot(const Tree &T0, int w, int order) {
  const int k = T0.k;
  std::vector<std::vector<int>> adj(k);
  for (int i = 0; i < k; ++i)
    if (T0.parent[i] >= 0) {
      adj[i].push_back(T0.parent[i]);
      adj[T0.parent[i]].push_back(i);
    }
  Tree T;
  T.k = k;
  T.root = w;
  T.parent.assign(k, -1);
  T.child.assign(k, {});
  std::vector<int> queue{w}, seen(k, 0);
  seen[w] = 1;
  for (size_t h = 0; h < queue.size(); ++h) {
    const int x = queue[h];
    std::vector<int> nb = adj[x];
    std::sort(nb.begin(), nb.end());
    for (int y : nb)
      if (!seen[y]) {
        seen[y] = 1;
        T.parent[y] = x;
        T.child[x].push_back(y);
        queue.push_back(y);
      }
  }
  T.size.assign(k, 1);
  for (int h = (int)queue.size() - 1; h > 0; --h) T.size[T.parent[queue[h]]] += T.size[queue[h]];
  if (order)
    for (int x = 0; x < k; ++x)
      std::stable_sort(T.child[x].begin(), T.child[x].end(), [&](int a, int b) {
        return order == 1 ? T.size[a] < T.size[b] : T.size[a] > T.size[b];
      });
  return T;
}

Plan plan_rooted(const Tree &T);

// Model cost of one colouring of a plan (bytes-equivalent, compressed layout):
// each distinct passive of size p >= 2 gathers (k-1)/k x C(k-1, p-1) entries
// per adjacency entry (+ 4 B index) and writes C(k-1, p) per vertex; the
// colour histogram reads 5 B per adjacency entry; each combine reads and
// writes its rows and performs C(k-1,t-1) C(t-1,a-1) FMAs (weighted as
// `fma_bytes` bytes each).
double plan_cost(const Plan &P, const PlanOpts &o) {
  const int k = o.kc > 0 ? o.kc : P.k;  // colour universe
  const double e = o.elem, d = o.avg_degree;
  double c = 0;
  bool hist = false;
  std::vector<char> seen(P.tables.size(), 0);
  for (const Step &st : P.steps) {
    if (st.p == 1) {
      hist = true;
    } else if (!seen[st.passive]) {
      seen[st.passive] = 1;
      c += d * (4.0 + (double)(k - 1) / k * binom(k - 1, st.p - 1) * e) + binom(k - 1, st.p) * e;
    }
    if (st.a > 1) {
      const double rows = binom(k - 1, st.a - 1) + (st.out >= 0 ? binom(k - 1, st.p) + binom(k - 1, st.t - 1) : 1);
      c += rows * e + (st.out >= 0 ? binom(k - 1, st.t - 1) * (double)binom(st.t - 1, st.a - 1) : binom(k - 1, st.a - 1)) *
                           o.fma_bytes;
    }
  }
  if (hist) c += d * 5.0;
  return c;
}

Plan make_plan(int k, const int32_t *parent, const PlanOpts *opts) {
  Tree T0 = load_tree(k, parent);
  Plan base = plan_rooted(T0);
  base.kc = opts && opts->kc > 0 ? opts->kc : k;
  if (!opts || !opts->auto_root || k <= 2) return base;
  Plan best = base;
  double best_cost = plan_cost(base, *opts);
  for (int w = 0; w < k; ++w)
    for (int order = 0; order < 3; ++order) {
      Plan p = plan_rooted(reroot(T0, w, order));
      const double c = plan_cost(p, *opts);
      if (c < best_cost * (1.0 - 1e-9)) {
        best = std::move(p);
        best_cost = c;
      }
    }
  // |Aut|, |Aut_rho| and the Table-3 quantities refer to the user's rooting
  best.aut = base.aut;
  best.aut_root = base.aut_root;
  best.memory = base.memory;
  best.computation = base.computation;
  best.user_root = base.root;
  best.kc = base.kc;
  return best;
}

Plan plan_rooted(const Tree &T) {
  const int k = T.k;
  Plan P;
  P.k = k;
  P.root = T.root;
  P.user_root = T.root;
  P.parent = T.parent;

  // full-subtree codes in the template's own rooting
  std::vector<std::string> full(k);
  std::function<void(int)> fc = [&](int x) {
    std::vector<std::string> cs;
    for (int c : T.child[x]) {
      fc(c);
      cs.push_back(full[c]);
    }
    std::sort(cs.begin(), cs.end());
    std::string s = "(";
    for (auto &c : cs) s += c;
    full[x] = s + ")";
  };
  fc(T.root);
  auto partial_code = [&](int x, int j) {
    std::vector<std::string> cs;
    for (int i = 0; i < j; ++i) cs.push_back(full[T.child[x][i]]);
    std::sort(cs.begin(), cs.end());
    std::string s = "(";
    for (auto &c : cs) s += c;
    return s + ")";
  };
  auto partial_size = [&](int x, int j) {
    int s = 1;
    for (int i = 0; i < j; ++i) s += T.size[T.child[x][i]];
    return s;
  };

  std::map<std::string, int> memo;
  std::function<int(int, int)> get = [&](int x, int j) -> int {
    if (j == 0) return -1;  // single vertex, implicit table
    std::string code = partial_code(x, j);
    auto it = memo.find(code);
    if (it != memo.end()) return it->second;
    int A = get(x, j - 1);
    int y = T.child[x][j - 1];
    int Pid = get(y, (int)T.child[y].size());
    int id = (int)P.tables.size();
    P.tables.push_back({partial_size(x, j), x, j, code});
    int t = partial_size(x, j), a = partial_size(x, j - 1);
    P.steps.push_back({t, a, t - a, A, Pid, id});
    memo[code] = id;
    return id;
  };

  if (k > 1) {
    int nr = (int)T.child[T.root].size();
    int A = get(T.root, nr - 1);
    int y = T.child[T.root][nr - 1];
    int Pid = get(y, (int)T.child[y].size());
    int a = partial_size(T.root, nr - 1);
    P.steps.push_back({k, a, k - a, A, Pid, -1});
  }

  P.full_table.assign(k, -1);
  for (int x = 0; x < k; ++x) {
    if (x == T.root) P.full_table[x] = -2;
    else if (!T.child[x].empty()) P.full_table[x] = memo.at(full[x]);
  }

  // liveness
  const int nt = (int)P.tables.size();
  P.table_last_use.assign(nt, -1);
  P.n_first_use.assign(nt, -1);
  P.n_last_use.assign(nt, -1);
  for (int s = 0; s < (int)P.steps.size(); ++s) {
    const Step &st = P.steps[s];
    if (st.active >= 0) P.table_last_use[st.active] = std::max(P.table_last_use[st.active], s);
    if (st.passive >= 0) {
      if (P.n_first_use[st.passive] < 0) {
        P.n_first_use[st.passive] = s;
        P.table_last_use[st.passive] = std::max(P.table_last_use[st.passive], s);
      }
      P.n_last_use[st.passive] = s;
    }
  }

  // automorphisms: |Aut_rho| = prod over vertices of prod over classes of
  // identical child subtrees of (multiplicity)!; |Aut| = |Aut_rho| x |orbit(rho)|.
  P.aut_root = 1;
  for (int x = 0; x < k; ++x) {
    std::map<std::string, int> mult;
    for (int c : T.child[x]) mult[full[c]]++;
    for (auto &kv : mult) P.aut_root *= factorial(kv.second);
  }
  std::vector<std::vector<int>> adj(k);
  for (int i = 0; i < k; ++i)
    if (T.parent[i] >= 0) {
      adj[i].push_back(T.parent[i]);
      adj[T.parent[i]].push_back(i);
    }
  std::string rc = rooted_code(adj, T.root, -1);
  int orbit = 0;
  for (int w = 0; w < k; ++w) orbit += rooted_code(adj, w, -1) == rc;
  P.aut = P.aut_root * orbit;

  // Table 3: memory = sum C(k,t), computation =
  // sum C(k,t) C(t,a) over the non-root sub-templates of the plan.
  for (const Step &st : P.steps)
    if (st.out >= 0) {
      P.memory += (double)binom(k, st.t);
      P.computation += (double)binom(k, st.t) * (double)binom(st.t, st.a);
    }
  return P;
}

}  // namespace cc
