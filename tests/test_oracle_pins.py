"""Pins for the CPU oracle (-m "not gpu"): every oracle function is checked
against something other than itself -- the paper's worked example, closed
forms, textbook test vectors, invariants, and a pure-Python brute force of the
definition on tiny inputs.  See DESIGN.md "Oracle pins".
"""
import itertools
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


# ---------------------------------------------------------------- helpers
def py_brute(g, parent, colors=None):
    """Definition of PAPER.md lines 86-92 / 105-108 written out with
    itertools: injective f with template edges -> graph edges (and colourful)."""
    k = len(parent)
    adj = [set(g.neighbors(v).tolist()) for v in range(g.n)]
    cnt = 0
    for img in itertools.permutations(range(g.n), k):
        if any(parent[x] >= 0 and img[parent[x]] not in adj[img[x]] for x in range(k)):
            continue
        if colors is not None and len({int(colors[v]) for v in img}) < k:
            continue
        cnt += 1
    return cnt


def increasing_parents(k):
    """All parent arrays with parent[i] < i, root 0: every rooted tree shape on k vertices."""
    if k == 1:
        yield [-1]
        return
    for choice in itertools.product(*[range(i) for i in range(1, k)]):
        yield [-1] + list(choice)


def all_graphs(n):
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    for mask in range(1 << len(pairs)):
        yield synth.from_edges(n, [p for b, p in enumerate(pairs) if mask >> b & 1])


def exact_dp(g, parent, colors):
    return oracle.dp_count(g, parent, colors, oracle.NUM_EXACT).total


# ---------------------------------------------------------------- colouring
def test_mix_matches_splitmix64_reference_outputs():
    for i, hexv in _rows("splitmix64.txt"):
        assert oracle.mix(int(i) * 0x9E3779B97F4A7C15) == int(hexv, 16)


def test_color_formula_and_distribution():
    n, k, seed = 100_000, 5, 7
    c = oracle.color(n, k, seed)
    # formula of reading C-2, retyped as a spot check on a handful of ids only
    s = oracle.mix(seed)
    for v in (0, 1, 2, 99_999):
        assert c[v] == ((oracle.mix(s ^ v) >> 32) * k) >> 32
    # uniform: every colour within 5 sigma of n/k (SPEC random_coloring example)
    counts = np.bincount(c, minlength=k)
    sigma = math.sqrt(n * (1 / k) * (1 - 1 / k))
    assert np.all(np.abs(counts - n / k) < 5 * sigma)
    assert np.array_equal(c, oracle.color(n, k, seed))          # deterministic
    assert not np.array_equal(c, oracle.color(n, k, seed + 1))  # seed matters
    assert np.all(oracle.color(50, 1, 3) == 0)                  # k = 1


# ---------------------------------------------------------------- brute force
def test_c_brute_force_matches_python_definition():
    rng = np.random.default_rng(0)
    for trial in range(40):
        n = int(rng.integers(3, 7))
        g = synth.gnp(n, float(rng.choice([0.3, 0.6, 0.9])), int(rng.integers(1 << 30)))
        k = int(rng.integers(1, min(n, 4) + 1))
        parent = list(next(itertools.islice(increasing_parents(k), int(rng.integers(math.factorial(k - 1))), None)))
        col = rng.integers(0, k, n).astype(np.uint8)
        assert oracle.brute_count(g, parent) == py_brute(g, parent)
        assert oracle.brute_count(g, parent, col) == py_brute(g, parent, col)


def test_spec_tiny_values():
    tri = synth.cycle(3)
    for name, par, cols, maps in _rows("spec_tiny.txt"):
        parent = [int(x) for x in par.split(",")]
        if cols == "-":
            assert oracle.brute_count(tri, parent) == int(maps), name
        else:
            col = np.array([int(x) for x in cols.split(",")], dtype=np.uint8)
            assert oracle.brute_count(tri, parent, col) == int(maps), name
            assert exact_dp(tri, parent, col) == int(maps), name


def test_aut_against_permutations_and_hand_values():
    # brute force over vertex permutations (definition of an automorphism), k <= 7
    for k in range(1, 7):
        for parent in itertools.islice(increasing_parents(k), 0, None, 7):
            edges = {frozenset((i, p)) for i, p in enumerate(parent) if p >= 0}
            perms = sum(1 for pm in itertools.permutations(range(k))
                        if {frozenset((pm[a], pm[b])) for a, b in map(tuple, edges)} == edges)
            assert oracle.aut(parent) == perms, parent
    # hand-derived: P5 reversal 2; 3-leg spiders 3! = 6; 12-tree: two swaps under
    # vertex 1 and one of its children pair = 8; perfect binary tree of depth 3: 2^7
    from synth import CONFIGS
    assert [oracle.aut(c.parent) for c in CONFIGS] == [2, 6, 6, 8, 128]


# ---------------------------------------------------------------- DP vs brute force
def test_dp_exhaustive_n4_all_trees_all_colourings():
    for g in all_graphs(4):
        for k in range(1, 5):
            for parent in increasing_parents(k):
                for cols in itertools.product(range(k), repeat=4):
                    col = np.array(cols, dtype=np.uint8)
                    assert exact_dp(g, parent, col) == oracle.brute_count(g, parent, col)


def test_dp_all_graphs_n5_random_colourings():
    rng = np.random.default_rng(5)
    for g in all_graphs(5):
        for k in range(2, 6):
            for parent in increasing_parents(k):
                col = rng.integers(0, k, 5).astype(np.uint8)
                assert exact_dp(g, parent, col) == oracle.brute_count(g, parent, col)


def test_dp_random_graphs_trees_up_to_7_and_any_root_position():
    rng = np.random.default_rng(11)
    for trial in range(60):
        k = int(rng.integers(2, 8))
        n = int(rng.integers(k, 11))
        g = synth.gnp(n, float(rng.choice([0.2, 0.5, 0.9])), int(rng.integers(1 << 30)))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, k)]
        # relabel template vertices so the root is not vertex 0 and parents may follow children
        perm = rng.permutation(k)
        inv = np.argsort(perm)
        relab = [-1] * k
        for x in range(k):
            relab[perm[x]] = -1 if parent[x] < 0 else int(perm[parent[x]])
        for par in (parent, relab):
            col = rng.integers(0, k, n).astype(np.uint8)
            assert exact_dp(g, par, col) == oracle.brute_count(g, par, col)
        del inv


@pytest.mark.parametrize("ci", [0, 1, 2, 3])
def test_dp_config_templates_on_12_vertex_graphs(ci):
    cfg = synth.CONFIGS[ci]
    rng = np.random.default_rng(ci)
    for p in (0.4, 0.8):
        g = synth.gnp(12, p, 100 + ci)
        col = rng.integers(0, cfg.k, 12).astype(np.uint8)
        assert exact_dp(g, cfg.parent, col) == oracle.brute_count(g, cfg.parent, col)


def test_dp_k15_template_sparse_graphs_and_G_equals_T():
    par = synth.CONFIGS[4].parent
    rng = np.random.default_rng(15)
    for n in (15, 17):
        g = synth.disjoint_union(synth.tree_graph(par), synth.gnp(n - 15 + 4, 0.5, n)) if n > 15 \
            else synth.tree_graph(par)
        col = rng.integers(0, 15, g.n).astype(np.uint8)
        assert exact_dp(g, par, col) == oracle.brute_count(g, par, col)
    # G = T with a bijective colouring: X = |Aut(T)| for every config template
    for cfg in synth.CONFIGS:
        g = synth.tree_graph(cfg.parent)
        col = rng.permutation(cfg.k).astype(np.uint8)
        assert exact_dp(g, cfg.parent, col) == oracle.aut(cfg.parent)


def test_dp_config0_equals_brute_force():
    cfg = synth.CONFIGS[0]
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, cfg.color_seed)
    x = exact_dp(g, cfg.parent, col)
    assert x == oracle.brute_count(g, cfg.parent, col)
    assert 0 < x < 2 ** 53
    # the float instantiations agree exactly in the integer regime
    assert oracle.dp_count(g, cfg.parent, col, oracle.NUM_DOUBLE).total == float(x)
    assert oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE).total == float(x)


# ---------------------------------------------------------------- closed forms
def _star(k):
    return [-1] + [0] * (k - 1)


def test_star_closed_forms_rmat():
    g = synth.rmat(11, 8, seed=3)
    deg = g.degrees()
    for k in (3, 4, 5):
        col = oracle.color(g.n, k, 40 + k)
        onehot = np.zeros((g.n, k), dtype=object)
        for v in range(g.n):
            for u in g.neighbors(v):
                onehot[v, col[u]] += 1
        want = 0
        for v in range(g.n):
            prod = 1
            for j in range(k):
                if j != col[v]:
                    prod *= int(onehot[v, j])
            want += prod
        want *= math.factorial(k - 1)
        assert exact_dp(g, _star(k), col) == want
    # exact maps of a star: sum_v (deg v)_(k-1) falling factorial = (k-1)! C(deg, k-1) (BJ)
    gs = synth.gnp(9, 0.5, 4)
    for k in (3, 4):
        want = sum(math.perm(int(d), k - 1) for d in gs.degrees())
        assert oracle.brute_count(gs, _star(k)) == want


def test_clique_closed_forms_every_entry():
    # K_n: X = k! prod_j cnt_j ;  D_x(v,S) = [c_v in S] (s-1)! prod_{j in S, j != c_v} cnt_j
    n = 18
    g = synth.clique(n)
    for cfg in synth.CONFIGS[:4]:
        k = cfg.k
        col = oracle.color(n, k, 5 + k)
        cnt = np.bincount(col, minlength=k)
        assert exact_dp(g, cfg.parent, col) == math.factorial(k) * math.prod(int(c) for c in cnt)
        sizes = oracle.subtree_sizes(cfg.parent)
        for x in range(k):
            s = sizes[x]
            tab = oracle.dp_count(g, cfg.parent, col, oracle.NUM_EXACT, keep_x=x).table
            subsets = [S for S in itertools.combinations(range(k), s)]
            # colex order: sort by the reversed tuple
            subsets.sort(key=lambda S: S[::-1])
            for v in range(n):
                want = [(math.factorial(s - 1) * math.prod(int(cnt[j]) - (1 if j == col[v] else 0)
                                                            for j in S if j != col[v]))
                        if col[v] in S else 0 for S in subsets]
                # neighbours exclude v itself: counts of colour j among N(v) = cnt_j - [j == c_v]
                assert np.array_equal(tab[v], np.array(want, dtype=np.float64)), (cfg.name, x, v)


def test_path_on_cycle_windows():
    rng = np.random.default_rng(3)
    for n, k in ((20, 4), (31, 5), (24, 6)):
        g = synth.cycle(n)
        parent = [-1] + list(range(k - 1))
        for _ in range(3):
            col = rng.integers(0, k, n).astype(np.uint8)
            win = sum(1 for i in range(n) if len({int(col[(i + j) % n]) for j in range(k)}) == k)
            assert exact_dp(g, parent, col) == 2 * win
        col = (np.arange(n) % k).astype(np.uint8)
        if n % k == 0:
            assert exact_dp(g, parent, col) == 2 * n


def test_sum_over_all_colourings_identity():
    # sum over all k^n colourings of X = k! k^(n-k) maps (each map colourful in k! k^(n-k) colourings)
    g = synth.gnp(6, 0.6, 9)
    for parent in ([-1, 0, 1], [-1, 0, 0], [-1, 0, 1, 1]):
        k = len(parent)
        tot = sum(exact_dp(g, parent, np.array(c, dtype=np.uint8))
                  for c in itertools.product(range(k), repeat=g.n))
        assert tot == math.factorial(k) * k ** (g.n - k) * oracle.brute_count(g, parent)


def test_invariants_monotone_additive_bounded():
    rng = np.random.default_rng(21)
    parent = [-1, 0, 0, 1]
    g = synth.gnp(10, 0.3, 1)
    h = synth.gnp(8, 0.5, 2)
    col = rng.integers(0, 4, g.n + h.n).astype(np.uint8)
    u = synth.disjoint_union(g, h)
    xg, xh = exact_dp(g, parent, col[:g.n]), exact_dp(h, parent, col[g.n:])
    assert exact_dp(u, parent, col) == xg + xh                     # additive over disjoint union
    assert xg <= oracle.brute_count(g, parent)                     # colourful <= all maps
    e = np.stack(g.edges(), 1).tolist()
    g2 = synth.from_edges(g.n, e + [(0, 9), (2, 7)])
    assert exact_dp(g2, parent, col[:g.n]) >= xg                   # monotone in edges
    # colour permutation invariance
    perm = rng.permutation(4).astype(np.uint8)
    assert exact_dp(g, parent, perm[col[:g.n]]) == xg
    # root / cut-order invariance: the same tree written with another root
    assert exact_dp(g, [1, 3, 0, -1], col[:g.n]) == xg  # path 3-1-0-2 rooted at 3


# ---------------------------------------------------------------- combine & estimator
def test_fig1b_partial_sum_is_6():
    rows = _rows("paper_fig1b.txt")
    k = 5

    def rank(S):  # colex = position among same-size subsets sorted by reversed tuple
        size = len(S)
        allS = sorted(itertools.combinations(range(k), size), key=lambda t: t[::-1])
        return allS.index(tuple(sorted(S)))

    A = np.zeros(math.comb(k, 2))
    N = np.zeros(math.comb(k, 3))
    want = None
    for kind, cols, val in rows:
        S = [int(c) for c in cols.split(",")]
        if kind == "A":
            A[rank(S)] = float(val)
        elif kind == "N":
            N[rank(S)] = float(val)
        else:
            want = float(val)
    T = oracle.combine_row(k, 2, 3, A, N)
    assert T[0] == want == 6.0


def test_estimator_scaling_spec_values_and_unbiasedness():
    # k=3, raw 6 -> 27 (|Aut| = 1 to isolate the k^k/k! factor); S:456 factor 3125/120
    assert oracle.estimate([6.0], 3, 1) == pytest.approx(27.0, rel=1e-15)
    assert oracle.estimate([120.0], 5, 1) == pytest.approx(3125.0, rel=1e-15)
    assert oracle.estimate([0.0, 0.0], 4, 2) == 0.0
    # statistical: the mean over colourings approaches copies = maps/|Aut| (within 4 s.e.)
    g = synth.gnp(14, 0.35, 8)
    parent = [-1, 0, 1, 0]
    k = 4
    aut_t = oracle.aut(parent)
    copies = oracle.brute_count(g, parent) / aut_t
    xs = [exact_dp(g, parent, oracle.color(g.n, k, s)) for s in range(400)]
    est = oracle.estimate(xs, k, aut_t)
    se = np.std(np.array(xs, dtype=float) * k ** k / math.factorial(k) / aut_t) / math.sqrt(len(xs))
    assert abs(est - copies) < 4 * se


def test_table3_intensity_values():
    """Table 3 restated from its definition (lines
    605-608): memory = sum C(k,t), computation = sum C(k,t) C(t,a) over the
    non-root, non-leaf sub-templates of a path rooted at an end (reading C-14)."""
    for name, par, mem, comp, inten in _rows("table3.txt"):
        k = len(par.split(","))
        subs = [(t, 1) for t in range(2, k)]  # path rooted at an end: steps (t; 1, t-1), C(t,1) splits
        m = sum(math.comb(k, t) for t, _ in subs)
        c = sum(math.comb(k, t) * math.comb(t, 1) for t, _ in subs)
        assert m == int(mem) and c == int(comp) and round(c / m, 1) == float(inten), name


def test_niter_spec_values():
    """Niter = ceil(c e^k ln(1/delta) / eps^2) (Alg. 1 line 3; SPEC.md
    lines 441-446 worked values)."""
    assert oracle.niter(0.5, 0.1, 3) == 185  # ceil(20.0855 x 2.3026 / 0.25)
    assert oracle.niter(0.5, 1.0, 3) == 1  # delta -> 1 clamps to 1
    for eps in (0.5, 0.3, 0.1):  # halving eps quadruples Niter up to the ceiling
        a, b = oracle.niter(eps, 0.05, 5), oracle.niter(eps / 2, 0.05, 5)
        assert 4 * a - 4 <= b <= 4 * a
    assert oracle.niter(0.5, 0.1, 3, c=2.0) == math.ceil(2 * math.exp(3) * math.log(10) / 0.25)


def test_median_of_means_spec_values():
    """Median of group means (Alg. 1 last line, lines 180-181; SPEC.md
    lines 455-463): groups of floor(N/t) in iteration order, remainder one per
    group from the front; mean of the two middle values for even t."""
    s3 = 27 / 6  # k = 3 scale k^k/k!, |Aut| = 1
    assert oracle.median_of_means([0, 0, 0, 100], 3, 1, 4) == 0.0  # S:461 outlier robustness
    assert oracle.median_of_means([7.0] * 9, 3, 1, 3) == pytest.approx(7 * s3, rel=1e-15)  # S:460 constant
    xs = [1.0, 2.0, 4.0, 8.0, 16.0]
    assert oracle.median_of_means(xs, 3, 1, 1) == pytest.approx(oracle.estimate(xs, 3, 1), rel=1e-15)
    # N = 5, t = 2: groups {1, 2, 4} and {8, 16}; even t -> mean of the two group means
    assert oracle.median_of_means(xs, 3, 1, 2) == pytest.approx(((7 / 3) + 12) / 2 * s3, rel=1e-15)
    # N = 7, t = 3: sizes 3, 2, 2 -> means 2, 4.5, 7 -> median 4.5 (|Aut| = 2 halves it)
    assert oracle.median_of_means([1, 2, 3, 4, 5, 6, 8], 3, 2, 3) == pytest.approx(4.5 * s3 / 2, rel=1e-15)
    with pytest.raises(oracle.OracleError):
        oracle.median_of_means([1.0], 3, 1, 2)


def test_more_colours_than_vertices_dp_equals_brute_force():
    """kc > k colours: the DP over the kc-colour universe, summed
    over every colour set of size k at the root, still counts exactly the
    colourful maps of the definition (distinct colours; PAPER.md lines
    105-108), which the brute force enumerates without any colour sets."""
    rng = np.random.default_rng(21)
    for trial in range(24):
        k = int(rng.integers(2, 6))
        kc = int(rng.integers(k, min(k + 5, 16) + 1))
        n = int(rng.integers(k, 14))
        g = synth.gnp(n, float(rng.choice([0.3, 0.6])), int(rng.integers(1 << 30)))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, k)]
        col = rng.integers(0, kc, n).astype(np.uint8)
        want = oracle.brute_count(g, parent, col)
        r = oracle.dp_count(g, parent, col, oracle.NUM_EXACT, want_root=True, colours=kc)
        assert r.total == want, (k, kc, parent)
        assert float(r.root.sum()) == float(want)
    # kc = k is the plain DP
    g = synth.gnp(10, 0.5, 3)
    col = oracle.color(g.n, 4, 7)
    assert oracle.dp_count(g, [-1, 0, 1, 1], col, colours=4).total == oracle.dp_count(g, [-1, 0, 1, 1], col).total


def test_more_colours_sum_over_all_colourings():
    """Summed over all kc^n colourings, X = kc!/(kc-k)! kc^(n-k) maps: each map
    is colourful for kc (kc-1) ... (kc-k+1) colourings of its k image vertices
    (the colourful probability of PAPER.md line 146 with kc colours)."""
    g = synth.gnp(5, 0.7, 11)
    parent = [-1, 0, 1]
    k, kc = 3, 4
    maps = oracle.brute_count(g, parent)
    total = 0
    for col in itertools.product(range(kc), repeat=g.n):
        total += oracle.dp_count(g, parent, np.array(col, np.uint8), colours=kc).total
    assert total == math.perm(kc, k) * kc ** (g.n - k) * maps


# ---------------------------------------------------------------- the root count at one vertex
def test_dp_root_at_sums_to_brute_force_and_equals_the_dp_root_row():
    """or_dp_root_at (the DP evaluated only within each template vertex's
    depth of v0): summed over every v0 it is the brute force of the
    definition -- the pin independent of the
    DP -- and at each v0 it is the full DP's per-vertex root D_root(v0, [k]);
    also on the subgraph induced by the ball of radius height(T) around v0
    (the locality the full-size sampled checks rely on)."""
    rng = np.random.default_rng(21)
    for trial in range(40):
        k = int(rng.integers(1, 8))
        n = int(rng.integers(max(k, 2), 12))
        g = synth.gnp(n, float(rng.choice([0.25, 0.5, 0.8])), int(rng.integers(1 << 30)))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, k)]
        perm = rng.permutation(k)
        relab = [-1] * k
        for x in range(k):
            relab[perm[x]] = -1 if parent[x] < 0 else int(perm[parent[x]])
        col = rng.integers(0, k, n).astype(np.uint8)
        per_v = [oracle.dp_root_at(g, relab, col, v) for v in range(n)]
        assert sum(per_v) == oracle.brute_count(g, relab, col), (relab, per_v)
        full = oracle.dp_count(g, relab, col, oracle.NUM_EXACT, want_root=True).root
        assert [float(x) for x in per_v] == full.tolist()
    # locality: the ball of radius height(T) around v0 carries the whole answer
    g = synth.rmat(9, 8, seed=4)
    for parent in (synth.CONFIGS[2].parent, synth.CONFIGS[4].parent):
        k = len(parent)
        depth = [0] * k
        for x in range(k):
            p = parent[x]
            while p >= 0:
                depth[x] += 1
                p = parent[p]
        h = max(depth)
        col = oracle.color(g.n, k, 8)
        full = oracle.dp_count(g, parent, col, oracle.NUM_EXACT, want_root=True).root
        for v0 in (0, 5, 100, 300):
            ball = {v0}
            frontier = {v0}
            for _ in range(h):
                frontier = {int(u) for w in frontier for u in g.neighbors(w)} - ball
                ball |= frontier
            verts = np.array(sorted(ball))
            idx = {int(v): i for i, v in enumerate(verts)}
            edges = [(idx[int(v)], idx[int(u)]) for v in verts for u in g.neighbors(int(v)) if int(u) in idx and u > v]
            sub = synth.from_edges(len(verts), edges)
            got = oracle.dp_root_at(sub, parent, col[verts], idx[v0])
            assert float(got) == full[v0], (parent, v0)
            assert oracle.dp_root_at(g, parent, col, v0) == got
