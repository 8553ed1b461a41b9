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

Plan make_plan(int k, const int32_t *parent) {
  Tree T = load_tree(k, parent);
  Plan P;
  P.k = k;
  P.root = T.root;
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
