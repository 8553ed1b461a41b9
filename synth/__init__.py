"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO colour-coding arithmetic (no colouring hash, no colour
sets, no counting): it only builds graphs (CSR) and the five workload recipes
of BASELINE.json `configs`, which stand in for the paper's datasets (PAPER.md
Table 2) and template figure (PAPER.md, lost).

Graphs come from the C generator `synth/gen.c` (counter-based, deterministic,
OpenMP); tiny structured graphs (cycle, clique, star, ...) are built here.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO + ".tmp", src])
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp = ctypes.c_void_p
        lib.synth_rmat.restype = vp
        lib.synth_rmat.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_uint64]
        lib.synth_er.restype = vp
        lib.synth_er.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64]
        lib.synth_from_edges.restype = vp
        lib.synth_from_edges.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp]
        lib.synth_graph_size.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        lib.synth_graph_copy.argtypes = [vp, vp, vp]
        lib.synth_graph_free.argtypes = [vp]
        lib.synth_uniform_u8.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, vp]
        _lib = lib
    return _lib


@dataclass
class Graph:
    """Simple undirected graph in CSR form: row_ptr int64[n+1], col int32[2m], rows sorted."""
    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def m(self) -> int:
        return self.nnz // 2

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def neighbors(self, v: int) -> np.ndarray:
        return self.col[self.row_ptr[v]:self.row_ptr[v + 1]]

    def edges(self):
        """Undirected edges (u < v) as two int32 arrays."""
        src = np.repeat(np.arange(self.n, dtype=np.int64), self.degrees())
        keep = src < self.col
        return src[keep].astype(np.int32), self.col[keep].astype(np.int32)


def _take(h, name) -> Graph:
    lib = _load()
    if not h:
        raise ValueError("synth: invalid generator arguments")
    n = ctypes.c_int64()
    nnz = ctypes.c_int64()
    lib.synth_graph_size(h, ctypes.byref(n), ctypes.byref(nnz))
    rp = np.empty(n.value + 1, dtype=np.int64)
    col = np.empty(max(nnz.value, 1), dtype=np.int32)[:nnz.value]
    lib.synth_graph_copy(h, rp.ctypes.data, col.ctypes.data if nnz.value else None)
    lib.synth_graph_free(h)
    return Graph(int(n.value), rp, col, name)


def rmat(scale: int, edge_factor: int, a=0.57, b=0.19, c=0.19, seed: int = 1) -> Graph:
    """R-MAT (BASELINE.json configs 1-4): 2^scale vertices, edge_factor*2^scale draws,
    symmetrised, deduplicated, self-loops removed."""
    h = _load().synth_rmat(scale, edge_factor, a, b, c, seed)
    return _take(h, f"rmat-s{scale}-ef{edge_factor}-seed{seed}")


def erdos_renyi(n: int, m: int, seed: int = 1) -> Graph:
    """G(n, m): m distinct edges drawn uniformly (BASELINE.json config 0)."""
    h = _load().synth_er(n, m, seed)
    return _take(h, f"er-{n}-{m}-seed{seed}")


def from_edges(n: int, edges) -> Graph:
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    eu = np.ascontiguousarray(e[:, 0], dtype=np.int32)
    ev = np.ascontiguousarray(e[:, 1], dtype=np.int32)
    if len(e) and (e.min() < 0 or e.max() >= n):
        raise ValueError("edge endpoint out of range")
    h = _load().synth_from_edges(n, len(e), eu.ctypes.data if len(e) else None,
                                 ev.ctypes.data if len(e) else None)
    return _take(h, "edges")


def cycle(n: int) -> Graph:
    return from_edges(n, [(i, (i + 1) % n) for i in range(n)])


def path(n: int) -> Graph:
    return from_edges(n, [(i, i + 1) for i in range(n - 1)])


def clique(n: int) -> Graph:
    return from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])


def star(leaves: int) -> Graph:
    return from_edges(leaves + 1, [(0, i) for i in range(1, leaves + 1)])


def gnp(n: int, p: float, seed: int) -> Graph:
    """Small G(n, p) via numpy's PCG64 (test graphs only)."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < p
    return from_edges(n, np.stack([iu[keep], ju[keep]], axis=1))


def tree_graph(parent) -> Graph:
    """The template itself as a graph (for G = T pins)."""
    k = len(parent)
    return from_edges(k, [(i, p) for i, p in enumerate(parent) if p >= 0])


def disjoint_union(g: Graph, h: Graph) -> Graph:
    eu, ev = g.edges()
    fu, fv = h.edges()
    e = np.concatenate([np.stack([eu, ev], 1), np.stack([fu + g.n, fv + g.n], 1)]).astype(np.int64)
    return from_edges(g.n + h.n, e)


def uniform_colors(n: int, k: int, seed: int) -> np.ndarray:
    """A seeded uniform colouring passed IN as data (for set_colors tests)."""
    out = np.empty(max(n, 1), dtype=np.uint8)[:n]
    if n:
        _load().synth_uniform_u8(n, k, seed, out.ctypes.data)
    return out


# --------------------------------------------------------------------------
# BASELINE.json configs (the five workloads).  `graph()` builds the input.
# --------------------------------------------------------------------------
@dataclass
class Config:
    idx: int
    name: str
    parent: list
    precision: str            # "fp64" | "fp32"
    graph_kind: str            # "er" | "rmat"
    graph_args: dict = field(default_factory=dict)
    color_seed: int = 2
    colorings: int = 1

    @property
    def k(self) -> int:
        return len(self.parent)

    def graph(self) -> Graph:
        if self.graph_kind == "er":
            return erdos_renyi(**self.graph_args)
        return rmat(**self.graph_args)


CONFIGS = [
    Config(0, "er1000-P5", [-1, 0, 1, 2, 3], "fp64", "er", dict(n=1000, m=5000, seed=1)),
    Config(1, "rmat16-spider7", [-1, 0, 0, 0, 1, 2, 3], "fp64", "rmat",
           dict(scale=16, edge_factor=16, seed=1)),
    Config(2, "rmat20-spider10", [-1, 0, 1, 2, 0, 4, 5, 0, 7, 8], "fp32", "rmat",
           dict(scale=20, edge_factor=16, seed=1), colorings=10),
    Config(3, "rmat23-tree12", [-1, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5], "fp32", "rmat",
           dict(scale=23, edge_factor=32, seed=1)),
    Config(4, "rmat24-bintree15", [-1] + [(i - 1) // 2 for i in range(1, 15)], "fp32", "rmat",
           dict(scale=24, edge_factor=64, seed=1)),
]


def scaled_twin(cfg: Config, scale: int, edge_factor: int | None = None) -> Config:
    """Same template and generator at a smaller R-MAT scale (oracle-sized)."""
    ga = dict(cfg.graph_args)
    if cfg.graph_kind != "rmat":
        raise ValueError("only R-MAT configs have twins")
    ga["scale"] = scale
    if edge_factor is not None:
        ga["edge_factor"] = edge_factor
    return Config(cfg.idx, f"{cfg.name}-twin-s{scale}", cfg.parent, cfg.precision, "rmat", ga,
                  cfg.color_seed, cfg.colorings)
