"""-m "not gpu": host-side logic of the product library (no GPU needed):
the C ABI loads and exports every symbol of include/cc.h; colex indexing,
split tables, the template planner and the 1D partition are checked against
definitions, the paper's Table 3, and the oracle's independent |Aut(T)|."""
import itertools
import math
import os
import re

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cc():
    import __graft_entry__
    __graft_entry__._product_build()
    import paper_1804_09764_b200 as cc
    return cc


def test_library_exports_every_header_symbol(cc):
    hdr = open(os.path.join(ROOT, "include", "cc.h")).read()
    declared = set(re.findall(r"\b(cc_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations found"
    from paper_1804_09764_b200 import _native
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)
    for name in declared:
        assert hasattr(_native.lib, name), name


def test_colex_rank_examples_and_bijection(cc):
    # SPEC colex examples: k=3, s=2: {0,1}->0, {0,2}->1, {1,2}->2
    assert [cc.cc_colex_rank(m) for m in (0b011, 0b101, 0b110)] == [0, 1, 2]
    assert cc.cc_colex_rank(0b11111) == 0  # full set has rank 0
    for k in (5, 9, 12):
        for s in range(0, k + 1):
            masks = sorted(m for m in range(1 << k) if bin(m).count("1") == s)  # colex = increasing mask
            assert [cc.cc_colex_rank(m) for m in masks] == list(range(len(masks)))
            assert [cc.cc_colex_unrank(s, r) for r in range(len(masks))] == masks
    # complement reverses colex order when t = k/2 (SURVEY 8(f) F3 check)
    k = 8
    masks = sorted(m for m in range(1 << k) if bin(m).count("1") == 4)
    full = (1 << k) - 1
    assert [cc.cc_colex_rank(full ^ m) for m in masks] == list(range(len(masks)))[::-1]


def test_split_tables_are_exactly_the_disjoint_splits(cc):
    for k, t, a in ((5, 3, 1), (7, 5, 3), (12, 7, 4), (10, 10, 7), (15, 8, 1)):
        tab = cc.cc_split_table(k, t, a)
        assert tab.shape == (math.comb(t, a), math.comb(k, t))
        sets = {s: sorted(m for m in range(1 << k) if bin(m).count("1") == s) for s in (t, a, t - a)}
        for r in range(0, math.comb(k, t), max(1, math.comb(k, t) // 50)):
            S = sets[t][r]
            pairs = {(sets[a][p & 0xFFFF], sets[t - a][p >> 16]) for p in tab[:, r].tolist()}
            want = {(X, S ^ X) for X in sets[a] if X & S == X}
            assert pairs == want


def test_plans_of_the_configs(cc):
    want = [
        [(2, 1, 1), (3, 1, 2), (4, 1, 3), (5, 1, 4)],
        [(2, 1, 1), (3, 1, 2), (5, 3, 2), (7, 5, 2)],
        [(2, 1, 1), (3, 1, 2), (4, 1, 3), (7, 4, 3), (10, 7, 3)],
        [(2, 1, 1), (3, 2, 1), (4, 1, 3), (7, 4, 3), (8, 1, 7), (3, 1, 2), (4, 3, 1), (12, 8, 4)],
        [(2, 1, 1), (3, 2, 1), (4, 1, 3), (7, 4, 3), (8, 1, 7), (15, 8, 7)],
    ]
    for cfg, w in zip(synth.CONFIGS, want):
        p = cc.cc_plan_template(cfg.parent)
        assert [(s["t"], s["a"], s["p"]) for s in p["steps"]] == w
        assert p["aut"] == oracle.aut(cfg.parent)
        # every step: t = a + p, the root step is last, tables used after being produced
        made = set()
        for i, s in enumerate(p["steps"]):
            assert s["t"] == s["a"] + s["p"]
            for tid in (s["active"], s["passive"]):
                assert tid == -1 or tid in made
            if s["out"] >= 0:
                made.add(s["out"])
            else:
                assert i == len(p["steps"]) - 1 and s["t"] == cfg.k


def test_table3_memory_and_computation(cc):
    # PAPER.md Table 3 (lines 587-596): u3-1 3/6 (intensity 2), u5-2 25/70 (2.8)
    for par, mem, comp in (([-1, 0, 1], 3, 6), ([-1, 0, 1, 2, 3], 25, 70)):
        p = cc.cc_plan_template(par)
        assert (p["memory"], p["computation"]) == (mem, comp)


def test_aut_matches_oracle_on_all_small_trees(cc):
    for k in range(1, 8):
        for choice in itertools.islice(itertools.product(*[range(i) for i in range(1, k)]), 0, None, 3):
            par = [-1] + list(choice)
            p = cc.cc_plan_template(par)
            assert p["aut"] == oracle.aut(par), par


def test_template_validation(cc):
    for bad in ([0, -1, 5], [-1, -1], [1, 0], [-1, 2, 1], list(range(-1, 16))):
        with pytest.raises(cc.CCError) as e:
            cc.cc_plan_template(bad)
        assert e.value.status in (cc.CC_ERR_TEMPLATE, cc.CC_ERR_ARG)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_invariants(cc, world):
    g = synth.rmat(12, 16, seed=2)
    deg = g.degrees()
    nz = set(np.nonzero(deg)[0].tolist())
    plans = [cc.cc_partition_plan(g.n, g.row_ptr, g.col, world, r) for r in range(world)]
    owned = np.concatenate([p["own_orig"] for p in plans])
    assert sorted(owned.tolist()) == sorted(nz)                     # disjoint cover of non-isolated
    owner = {int(v): r for r, p in enumerate(plans) for v in p["own_orig"]}
    adj_total = sum(int(deg[p["own_orig"]].sum()) for p in plans)
    assert adj_total == g.nnz
    loads = [int(deg[p["own_orig"]].sum()) + 16 * len(p["own_orig"]) for p in plans]
    assert max(loads) <= 1.25 * (sum(loads) / world) + int(deg.max())   # balanced
    for r, p in enumerate(plans):
        n_own = len(p["own_orig"])
        ids = np.concatenate([p["own_orig"], p["halo_orig"]])
        # the local CSR is the global adjacency, relabelled
        for i in range(0, n_own, max(1, n_own // 64)):
            v = p["own_orig"][i]
            loc = p["col"][p["rp"][i]:p["rp"][i + 1]]
            assert sorted(ids[loc].tolist()) == sorted(g.neighbors(v).tolist())
        # halo rows come from the peers, grouped; each peer's send list matches
        for q in range(world):
            recv = p["halo_orig"][p["recv_off"][q]:p["recv_off"][q + 1]]
            assert all(owner[int(v)] == q for v in recv)
            pq = plans[q]
            sent = pq["own_orig"][pq["send_idx"][pq["send_off"][r]:pq["send_off"][r + 1]]]
            assert np.array_equal(sent, recv)
        # hubs first within the rank
        d = deg[p["own_orig"]]
        assert np.all(d[:-1] >= d[1:])


def test_median_of_means_and_niter_match_the_oracle(cc):
    """The library's host-side estimator pieces against the oracle's (both
    pinned to PAPER.md Alg. 1 / SPEC.md worked values in test_oracle_pins)."""
    rng = np.random.default_rng(3)
    for n in (1, 2, 5, 7, 10, 33):
        xs = rng.integers(0, 10 ** 6, n).astype(np.float64)
        for t in sorted({1, 2, 3, n // 2 or 1, n}):
            if t > n:
                continue
            for k, aut in ((3, 1), (7, 6), (12, 8)):
                got = cc.cc_median_of_means(xs, k, aut, t)
                assert got == pytest.approx(oracle.median_of_means(xs, k, aut, t), rel=1e-15), (n, t, k)
    for eps, delta, k in ((0.5, 0.1, 3), (0.1, 0.01, 7), (0.05, 0.5, 12), (0.5, 1.0, 3)):
        assert cc.cc_niter(eps, delta, k) == oracle.niter(eps, delta, k)
    with pytest.raises(cc.CCError):
        cc.cc_median_of_means([1.0], 3, 1, 2)
    with pytest.raises(cc.CCError):
        cc.cc_niter(0.0, 0.1, 3)


@pytest.mark.parametrize("K,ts,as_", [(11, 8, 5), (14, 6, 3), (9, 6, 3), (8, 5, 2)])
def test_zblock_cover_computes_the_split_sum(cc, K, ts, as_):
    """The Z-block cover (register-blocked combine) covers every output set
    exactly once, and evaluating the combine through it (each block: its
    active sets x its passive sets, outputs Z minus one colour) equals the
    direct split sum of Eq. 1 over the split table, on random rows."""
    ps = ts - as_
    tab = cc.cc_zblock_table(K, ts, as_)
    na, nn, zs = math.comb(ts + 1, as_), math.comb(ts + 1, ps), ts + 1
    owned = tab[:, na + nn:na + nn + zs].ravel()
    owned = owned[owned != 0xFFFF]
    assert sorted(owned.tolist()) == list(range(math.comb(K, ts)))
    rng = np.random.default_rng(5)
    A = rng.random(math.comb(K, as_))
    N = rng.random(math.comb(K, ps))
    split = cc.cc_split_table(K, ts, as_)  # [q][r] = rank(X) | rank(Y) << 16
    direct = np.sum(A[split & 0xFFFF] * N[split >> 16], axis=0)
    local_sets = [c for c in itertools.combinations(range(zs), as_)]
    local_sets.sort(key=lambda s: s[::-1])  # colex order
    local_p = sorted(itertools.combinations(range(zs), ps), key=lambda s: s[::-1])
    pidx = {s: i for i, s in enumerate(local_p)}
    got = np.full(math.comb(K, ts), np.nan)
    for row in tab:
        acc = np.zeros(zs)
        for a, X in enumerate(local_sets):
            for z in range(zs):
                if z in X:
                    continue
                Y = tuple(sorted(set(range(zs)) - set(X) - {z}))
                acc[z] += A[row[a]] * N[row[na + pidx[Y]]]
        for z in range(zs):
            if row[na + nn + z] != 0xFFFF:
                got[row[na + nn + z]] = acc[z]
    assert np.allclose(got, direct, rtol=1e-12)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_exchange_model(cc, world):
    """The cost model behind CC_EXCHANGE_AUTO (Alg. 3 and the
    pipeline analysis, lines 326-341, 420-441), recomputed here from the
    partition plan: grouped = max(all halo rows over the link, local part) +
    one remote pass; ring = world - 1 steps in the order rank - 1, rank - 2,
    ..., each remote pass starting once its rows are in and the previous
    pass is done.  With two ranks the schedules coincide."""
    g = synth.rmat(12, 16, seed=2)
    w = 512.0
    for r in range(world):
        m = cc.cc_exchange_model(g.n, g.row_ptr, g.col, world, r, row_bytes=w)
        p = cc.cc_partition_plan(g.n, g.row_ptr, g.col, world, r)
        link, gbps, step = m["link_bps"], m["gather_bps"], 20e-6
        n_own = len(p["own_orig"])
        rp, col = p["rp"], p["col"]
        # owner of each halo row from recv_off
        halo_owner = np.repeat(np.arange(world), np.diff(p["recv_off"]))
        nnz = np.zeros(world)
        items = np.zeros(world)
        local = 0
        items_remote = 0
        for i in range(n_own):
            nb = col[rp[i]:rp[i + 1]]
            local += int((nb < n_own).sum())
            rem = nb[nb >= n_own] - n_own
            items_remote += len(rem) > 0
            cnt = np.bincount(halo_owner[rem], minlength=world)
            nnz += cnt
            items += cnt > 0

        def gather(e, t):
            return (e * (4 + w) + t * 2 * w) / gbps
        halo = np.diff(p["recv_off"]) * w / link
        grouped = max(halo.sum() + step, gather(local, 0)) + gather(nnz.sum(), items_remote)
        t, comm = gather(local, 0), 0.0
        for s in range(1, world):
            src = (r - s) % world
            comm += step + halo[src]
            t = max(t, comm) + gather(nnz[src], items[src])
        assert m["grouped_s"] == pytest.approx(grouped, rel=1e-9)
        assert m["ring_s"] == pytest.approx(t, rel=1e-9)
        if world == 2:
            assert m["ring_s"] == pytest.approx(m["grouped_s"], rel=1e-12)
    with pytest.raises(cc.CCError):
        cc.cc_exchange_model(g.n, g.row_ptr, g.col, 1, 0)


def test_no_fallback_without_the_library(tmp_path):
    """The product path fails loudly: the package without libcc.so raises
    ImportError (there is no CPU fallback), and without a GPU cc_create
    reports a CUDA error instead of computing anything."""
    import shutil
    import subprocess
    import sys
    pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1804_09764_b200")
    dst = tmp_path / "paper_1804_09764_b200"
    dst.mkdir()
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            shutil.copy(os.path.join(pkg, f), dst / f)
    r = subprocess.run([sys.executable, "-c", "import paper_1804_09764_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr and "not built" in r.stderr


def test_create_without_a_gpu_is_an_error(cc):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(cc.CCError) as e:
        cc.cc_create(device=0)
    assert e.value.status == cc.CC_ERR_CUDA


def test_bench_updates_match_the_library_plan(cc):
    """bench.py's U (pure Python, so that the oracle arm never loads the
    product) equals the distinct-passive count of the library's own
    fixed-root plan, for the five configs and random trees."""
    import bench
    rng = np.random.default_rng(3)
    parents = [c.parent for c in synth.CONFIGS]
    for _ in range(40):
        k = int(rng.integers(2, 13))
        parents.append([-1] + [int(rng.integers(0, i)) for i in range(1, k)])
    for parent in parents:
        k = len(parent)
        plan = cc.cc_plan_template(parent)
        seen, u = set(), 0
        for s in plan["steps"]:
            key = s["passive"] if s["p"] > 1 else "leaf"
            if key not in seen:
                seen.add(key)
                u += math.comb(k, s["p"])
        assert bench.updates_per_entry(parent) == u, parent


def test_reference_arm_does_not_load_the_product():
    import subprocess
    import sys
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', '0', '--steps', '1', "
            "'--warmup', '1']; runpy.run_path('bench.py', run_name='__main__'); "
            "assert 'paper_1804_09764_b200' not in sys.modules; "
            "maps = open('/proc/self/maps').read(); assert 'libcc.so' not in maps, 'libcc.so mapped'")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert '"impl": "reference"' in r.stdout


def test_bench_self_launches_n_ranks():
    """`bench.py --gpus 2` with no torchrun environment starts 2 ranks itself
    (torch.distributed.run on 127.0.0.1); the reference arm needs no GPU, so
    the launch is checked here: rank 0 alone prints the line, n_gpus = 2.  Our
    arm refuses to run when fewer GPUs than --gpus are visible."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--config", "0",
                        "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "0", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    import torch
    if torch.cuda.device_count() < 2:
        assert r.returncode == 2 and "CUDA device" in r.stderr
