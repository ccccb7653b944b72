"""Seeded synthetic inputs for the five BASELINE.json configurations.

Mesh and rest-data rules restate the reference so the GPU path, the C oracle and the
reference driver (oracle/ref_driver.cpp) all see bit-identical inputs:

* Kuhn 6-tet hex split -- /root/reference/proj/scenes/meshes/cube_2.tet:29-40
  (node id = (i*(n+1)+j)*(n+1)+k, hexes visited i, j, k with k fastest).
* quadratic edge nodes -- scene.hpp:909-932 (`expand_quadratic`, edge order
  {01,12,20,03,13,23}, new nodes appended in first-seen order).
* cloth diagonal rule -- scenes/meshes/cloth_8.tri:83-90; rest frame Dm2inv/area --
  scene.hpp:783-805; interior-edge flaps -- mesh_io.hpp:170-189; bending Q --
  energies.hpp:684-736; lumped mass -- scene.hpp:596-604.
* Lame parameters -- energies.hpp:23-30.

RNG: numpy PCG64 seeded with 0x5eed5eed + config index (SURVEY Appendix B7 leaves the
generator open; the committed golden fixtures pin the draws). Draws are node-major,
component-minor. No public dataset is involved: every config is synthetic by definition.
"""
from __future__ import annotations

import dataclasses
import os
from typing import Dict, Optional

import numpy as np

SEED_BASE = 0x5EED5EED


def lame_from_young_poisson(young: float, poisson: float):
    """energies.hpp:23-30 (same operation order)."""
    mu = young / (2.0 * (1.0 + poisson))
    lam = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson))
    return mu, lam


# --------------------------------------------------------------------------- meshes

def kuhn_grid(n: int):
    """(n+1)^3 nodes on [0,1]^3, 6 n^3 positively oriented tets (cube_2.tet:29-40)."""
    m = n + 1
    i, j, k = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    X = np.stack([i / n, j / n, k / n], axis=-1).reshape(-1, 3).astype(np.float64)
    hi, hj, hk = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    hi, hj, hk = hi.ravel(), hj.ravel(), hk.ravel()

    def v(a, b, c):
        return ((hi + a) * m + (hj + b)) * m + (hk + c)

    v000, v100, v110, v111 = v(0, 0, 0), v(1, 0, 0), v(1, 1, 0), v(1, 1, 1)
    v101, v010, v011, v001 = v(1, 0, 1), v(0, 1, 0), v(0, 1, 1), v(0, 0, 1)
    tets = np.stack([
        np.stack([v000, v100, v110, v111], 1),
        np.stack([v000, v101, v100, v111], 1),
        np.stack([v000, v110, v010, v111], 1),
        np.stack([v000, v010, v011, v111], 1),
        np.stack([v000, v001, v101, v111], 1),
        np.stack([v000, v011, v001, v111], 1),
    ], axis=1).reshape(-1, 4).astype(np.int64)
    return X, tets


TET10_EDGES = ((0, 1), (1, 2), (2, 0), (0, 3), (1, 3), (2, 3))


def expand_quadratic(tets: np.ndarray, X: np.ndarray):
    """scene.hpp:909-932: 10-node tets, edge nodes appended in first-seen order."""
    ne = tets.shape[0]
    a = np.stack([tets[:, e[0]] for e in TET10_EDGES], 1).ravel()
    b = np.stack([tets[:, e[1]] for e in TET10_EDGES], 1).ravel()
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    key = lo * (X.shape[0] + 1) + hi
    uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")          # unique keys in first-seen order
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    nv = X.shape[0]
    new_id = nv + rank[inv]
    ea, eb = a[first[order]], b[first[order]]
    mid = 0.5 * (X[ea] + X[eb])
    Xq = np.concatenate([X, mid], 0)
    conn = np.concatenate([tets, new_id.reshape(ne, 6)], 1).astype(np.int64)
    return Xq, conn


def signed_tet_volume(X: np.ndarray, t: np.ndarray) -> np.ndarray:
    """energies.hpp:323-334 `tet_rest_volume` operation order (det / 6)."""
    p0, p1, p2, p3 = X[t[:, 0]], X[t[:, 1]], X[t[:, 2]], X[t[:, 3]]
    e1, e2, e3 = p1 - p0, p2 - p0, p3 - p0
    det = (e1[:, 0] * (e2[:, 1] * e3[:, 2] - e2[:, 2] * e3[:, 1])
           - e1[:, 1] * (e2[:, 0] * e3[:, 2] - e2[:, 2] * e3[:, 0])
           + e1[:, 2] * (e2[:, 0] * e3[:, 1] - e2[:, 1] * e3[:, 0]))
    return det / 6.0


def lumped_mass(X: np.ndarray, conn: np.ndarray, density: float) -> np.ndarray:
    """scene.hpp:596-604: element mass density*V/npe added to each node, element order."""
    npe = conn.shape[1]
    vol = signed_tet_volume(X, conn[:, :4])
    mass = np.zeros(X.shape[0])
    contrib = density * vol / float(npe)
    for k in range(npe):                      # ascending element order per node
        np.add.at(mass, conn[:, k], contrib)
    return mass


def cloth_grid(N: int):
    """N x N node sheet on [0,1]^2, cloth_8.tri diagonal rule."""
    h = 1.0 / (N - 1)
    i, j = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    X = np.stack([i * h, j * h, np.zeros_like(i, dtype=np.float64)], -1).reshape(-1, 3)
    qi, qj = np.meshgrid(np.arange(N - 1), np.arange(N - 1), indexing="ij")
    qi, qj = qi.ravel(), qj.ravel()
    a = qi * N + qj
    even = ((qi + qj) % 2) == 0
    t1 = np.where(even[:, None], np.stack([a, a + N, a + N + 1], 1), np.stack([a, a + N, a + 1], 1))
    t2 = np.where(even[:, None], np.stack([a, a + N + 1, a + 1], 1), np.stack([a + N, a + N + 1, a + 1], 1))
    tris = np.stack([t1, t2], 1).reshape(-1, 3).astype(np.int64)
    return X.astype(np.float64), tris, h


def _dot(a, b):
    return a[..., 0] * b[..., 0] + a[..., 1] * b[..., 1] + a[..., 2] * b[..., 2]


def _cross(a, b):
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], -1)


def cloth_rest_frames(X: np.ndarray, tris: np.ndarray):
    """scene.hpp:783-805 (Dm2 = [[L1, t], [0, h]], inverse row-major; area = L1*h/2)."""
    E1 = X[tris[:, 1]] - X[tris[:, 0]]
    E2 = X[tris[:, 2]] - X[tris[:, 0]]
    L1 = np.sqrt(_dot(E1, E1))
    td = _dot(E1, E2) / L1
    P = E2 - (td / L1)[:, None] * E1
    h = np.sqrt(_dot(P, P))
    dmi = np.stack([1.0 / L1, -td / (L1 * h), np.zeros_like(L1), 1.0 / h], 1)
    area = 0.5 * L1 * h
    return dmi, area


def interior_edge_flaps(tris: np.ndarray) -> np.ndarray:
    """mesh_io.hpp:170-189: one flap (e0, e1, w0, w1) per edge with exactly two wings,
    edges in lexicographic (min, max) order, wings in encounter order."""
    ne = tris.shape[0]
    a = np.stack([tris[:, 0], tris[:, 1], tris[:, 2]], 1).ravel()
    b = np.stack([tris[:, 1], tris[:, 2], tris[:, 0]], 1).ravel()
    w = np.stack([tris[:, 2], tris[:, 0], tris[:, 1]], 1).ravel()
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    seq = np.arange(3 * ne)
    order = np.lexsort((seq, hi, lo))
    lo, hi, w = lo[order], hi[order], w[order]
    start = np.ones(lo.size, bool)
    start[1:] = (lo[1:] != lo[:-1]) | (hi[1:] != hi[:-1])
    gid = np.cumsum(start) - 1
    counts = np.bincount(gid)
    first = np.flatnonzero(start)
    keep = counts == 2
    f = first[keep]
    return np.stack([lo[f], hi[f], w[f], w[f + 1]], 1).astype(np.int64)


def bending_Q(X: np.ndarray, flaps: np.ndarray) -> np.ndarray:
    """energies.hpp:684-736 `precompute_bending_Q`, vectorised, same operation order."""
    X0, X1, X2, X3 = (X[flaps[:, k]] for k in range(4))

    def norm(v):
        return np.sqrt(_dot(v, v))

    def cot(u, v):
        s = norm(_cross(u, v))
        if np.any(s <= 0.0):
            raise ValueError("bending precompute: degenerate flap triangle")
        return _dot(u, v) / s

    c01 = cot(X1 - X0, X2 - X0)
    c02 = cot(X0 - X1, X2 - X1)
    c03 = cot(X1 - X0, X3 - X0)
    c04 = cot(X0 - X1, X3 - X1)
    A1 = 0.5 * norm(_cross(X1 - X0, X2 - X0))
    A2 = 0.5 * norm(_cross(X1 - X0, X3 - X0))
    kappa = np.stack([c02 + c04, c01 + c03, -(c01 + c02), -(c03 + c04)], 1)
    scale = 3.0 / (A1 + A2)
    Q = np.zeros((flaps.shape[0], 12, 12))
    for a in range(4):
        for c in range(4):
            v = scale * kappa[:, a] * kappa[:, c]
            for r in range(3):
                Q[:, 3 * a + r, 3 * c + r] = v
    return Q.reshape(-1, 144)


def random_rotations(rng, n):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
        np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
        np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1),
    ], 1)


def point_triangle_pairs(rng, x: np.ndarray, n_pairs: int, h: float, d_hat: float):
    """SURVEY 8(d) c5 / Appendix B4 offset form. Returns (pairs int64 [P,4] = (p,a,b,c),
    offsets float64 [P,12]) such that q_k = x[idx_k] + off_k realises a triangle with
    aspect ratio <= 10 and edges ~h, and a point projecting strictly inside it at
    distance d = d_hat * 10^(-4u) on the side of n = (b-a) x (c-a)."""
    nn = x.shape[0]
    idx = np.empty((n_pairs, 4), np.int64)
    # 4 distinct uniform nodes per pair (rejection on collisions)
    todo = np.arange(n_pairs)
    while todo.size:
        cand = rng.integers(0, nn, size=(todo.size, 4))
        s = np.sort(cand, 1)
        ok = np.all(s[:, 1:] != s[:, :-1], 1)
        idx[todo[ok]] = cand[ok]
        todo = todo[~ok]
    # local triangle A=(0,0), B=(L,0), C=(cx,cy) with aspect ratio <= 10
    L = np.empty(n_pairs); cx = np.empty(n_pairs); cy = np.empty(n_pairs)
    todo = np.arange(n_pairs)
    while todo.size:
        m = todo.size
        Lt = h * rng.uniform(0.5, 1.5, m)
        cxt = Lt * rng.uniform(-0.25, 1.25, m)
        cyt = h * rng.uniform(0.1, 1.5, m)
        e2 = np.maximum.reduce([Lt * Lt, cxt * cxt + cyt * cyt, (cxt - Lt) ** 2 + cyt * cyt])
        ar = e2 / (Lt * cyt)        # longest^2 / (2 * area)
        ok = ar <= 10.0
        L[todo[ok]] = Lt[ok]; cx[todo[ok]] = cxt[ok]; cy[todo[ok]] = cyt[ok]
        todo = todo[~ok]
    bary = rng.uniform(0.05, 1.0, size=(n_pairs, 3))
    bary /= bary.sum(1, keepdims=True)
    fx = bary[:, 1] * L + bary[:, 2] * cx
    fy = bary[:, 2] * cy
    d = d_hat * 10.0 ** (-4.0 * rng.uniform(0.0, 1.0, n_pairs))
    loc = np.zeros((n_pairs, 4, 3))
    loc[:, 0] = np.stack([fx, fy, d], 1)            # p
    loc[:, 2, 0] = L                                # b
    loc[:, 3, 0] = cx; loc[:, 3, 1] = cy            # c
    R = random_rotations(rng, n_pairs)
    geo = np.einsum("pij,pkj->pki", R, loc) + x[idx[:, 1]][:, None, :]
    off = (geo - x[idx]).reshape(n_pairs, 12)
    return idx, off, d


# --------------------------------------------------------------------------- configs

@dataclasses.dataclass
class Case:
    """One synthetic assembly workload. Arrays follow the reference registration:
    x (the only dof array, n x 3), rest (n x 3), per-energy connectivity and data."""
    name: str
    kind: str                      # tet4 | tet10 | cloth | contact
    x: np.ndarray
    X: np.ndarray
    conn: np.ndarray
    params: Dict[str, float]
    extra: Dict[str, np.ndarray] = dataclasses.field(default_factory=dict)

    @property
    def n_nodes(self) -> int:
        return self.x.shape[0]

    def n_elements(self) -> int:
        if self.kind == "cloth":
            return self.conn.shape[0] + self.extra["flaps"].shape[0]
        if self.kind == "contact":
            return self.conn.shape[0] + self.extra["pairs"].shape[0] + self.x.shape[0]
        return self.conn.shape[0]

    def write_case_dir(self, path: str) -> None:
        """Inputs for oracle/_ref/ref_driver (raw little-endian binaries + manifest)."""
        os.makedirs(path, exist_ok=True)
        self.x.astype(np.float64).tofile(os.path.join(path, "x.f64"))
        self.X.astype(np.float64).tofile(os.path.join(path, "X.f64"))
        self.conn.astype(np.int64).tofile(os.path.join(path, "conn.i64"))
        kind_map = {"pairs": "pairs.i64", "offsets": "offsets.f64", "mass": "mass.f64",
                    "x_prev": "x_prev.f64", "v": "v.f64"}
        for k, fn in kind_map.items():
            if k in self.extra:
                self.extra[k].tofile(os.path.join(path, fn))
        with open(os.path.join(path, "manifest.txt"), "w") as f:
            f.write(f"kind {self.kind}\n")
            for k, v in self.params.items():
                f.write(f"{k} {float(v)!r}\n")


NH_YOUNG, NH_POISSON = 1e5, 0.4


def tet4_case(n: int = 20, seed: int = SEED_BASE + 1, stretch: float = 1.2,
              noise: Optional[float] = 0.02, rel_noise: Optional[float] = None,
              name: str = "c1") -> Case:
    """Configs 1 (n=20, x = 1.2 stretch + U(+-0.02)) and 2 (n=100, x = X + U(+-0.3h))."""
    X, tets = kuhn_grid(n)
    rng = np.random.default_rng(seed)
    x = X.copy()
    x[:, 0] *= stretch
    amp = noise if rel_noise is None else rel_noise / n
    x += rng.uniform(-amp, amp, size=X.shape)
    mu, lam = lame_from_young_poisson(NH_YOUNG, NH_POISSON)
    return Case(name, "tet4", x, X, tets, {"mu": mu, "lambda": lam})


def hash_uniform(ids: np.ndarray, seed: int) -> np.ndarray:
    """Counter-based uniform [0, 1) draws (splitmix64 of seed + id): a node's noise depends only
    on its global id, so every rank of a sharded run regenerates the same values."""
    with np.errstate(over="ignore"):
        z = (np.asarray(ids, dtype=np.uint64) + np.uint64(seed)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


@dataclasses.dataclass
class SlabCase:
    """One rank's part of a slab-decomposed Kuhn-grid problem (owner computes).

    The global grid has world*n x n x n hexes on [0, world] x [0, 1]^2 (h = 1/n), node id
    (i*(n+1) + j)*(n+1) + k. Rank r owns node planes [r*n, (r+1)*n) (the last rank also the
    final plane) and the hexes whose first node v000 it owns, i.e. hex planes [r*n, (r+1)*n);
    it also evaluates the ghost hex plane r*n - 1 whose tets touch its first owned node plane,
    so its owned block rows are complete without any exchange. Local nodes are the planes
    [lo_hex, (r+1)*n], in global id order."""
    case: Case                 # local nodes, conn = own tets then ghost tets (local ids)
    n_own: int                 # own tets (first n_own rows of case.conn)
    row_lo: int                # owned block rows [row_lo, row_hi) in the local numbering
    row_hi: int
    global_ids: np.ndarray     # local node -> global node id


def _kuhn_x_range(n: int, hex_lo: int, own_lo: int, hex_hi: int, seed: int, rel_noise: float):
    """Hex planes [hex_lo, hex_hi) of the x-extended Kuhn grid (n x n hexes per plane), local
    nodes = planes [hex_lo, hex_hi]; tets of [own_lo, hex_hi) first, then of [hex_lo, own_lo)."""
    m = n + 1
    h = 1.0 / n
    planes = np.arange(hex_lo, hex_hi + 1)
    pi, pj, pk = np.meshgrid(planes, np.arange(m), np.arange(m), indexing="ij")
    gid = ((pi * m + pj) * m + pk).ravel().astype(np.int64)
    X = np.stack([pi.ravel() * h, pj.ravel() * h, pk.ravel() * h], 1).astype(np.float64)
    u = hash_uniform(gid[:, None] * 3 + np.arange(3)[None, :], seed)
    x = X + (2.0 * u - 1.0) * (rel_noise * h)

    def tets_of(hx):
        hi, hj, hk = np.meshgrid(hx - hex_lo, np.arange(n), np.arange(n), indexing="ij")
        hi, hj, hk = hi.ravel(), hj.ravel(), hk.ravel()

        def v(a, b, c):
            return ((hi + a) * m + (hj + b)) * m + (hk + c)

        v000, v100, v110, v111 = v(0, 0, 0), v(1, 0, 0), v(1, 1, 0), v(1, 1, 1)
        v101, v010, v011, v001 = v(1, 0, 1), v(0, 1, 0), v(0, 1, 1), v(0, 0, 1)
        return np.stack([np.stack([v000, v100, v110, v111], 1), np.stack([v000, v101, v100, v111], 1),
                         np.stack([v000, v110, v010, v111], 1), np.stack([v000, v010, v011, v111], 1),
                         np.stack([v000, v001, v101, v111], 1), np.stack([v000, v011, v001, v111], 1)],
                        axis=1).reshape(-1, 4).astype(np.int64)

    own = tets_of(np.arange(own_lo, hex_hi))
    ghost = tets_of(np.arange(hex_lo, own_lo))
    return x, X, own, ghost, gid


def tet4_slab_case(n: int, world: int, rank: int, seed: int = SEED_BASE + 2, rel_noise: float = 0.3) -> SlabCase:
    """Config-2 material and noise amplitude on a world-times-longer grid, this rank's slab."""
    m = n + 1
    hex_lo = rank * n - (1 if rank > 0 else 0)
    hex_hi = (rank + 1) * n
    x, X, own, ghost, gid = _kuhn_x_range(n, hex_lo, rank * n, hex_hi, seed, rel_noise)
    mu, lam = lame_from_young_poisson(NH_YOUNG, NH_POISSON)
    case = Case(f"c2slab{rank}of{world}", "tet4", x, X, np.concatenate([own, ghost]), {"mu": mu, "lambda": lam})
    row_lo = (rank * n - hex_lo) * m * m
    row_hi = (hex_hi - hex_lo + (1 if rank == world - 1 else 0)) * m * m
    return SlabCase(case, own.shape[0], row_lo, row_hi, gid)


def tet4_global_slab_case(n: int, world: int, seed: int = SEED_BASE + 2, rel_noise: float = 0.3) -> Case:
    """The whole world*n x n x n problem of tet4_slab_case in one piece (tests)."""
    x, X, own, _, _ = _kuhn_x_range(n, 0, 0, world * n, seed, rel_noise)
    mu, lam = lame_from_young_poisson(NH_YOUNG, NH_POISSON)
    return Case(f"c2slab_global{world}", "tet4", x, X, own, {"mu": mu, "lambda": lam})


def config1(n: int = 20) -> Case:
    return tet4_case(n, SEED_BASE + 1, 1.2, 0.02, None, "c1")


def config2(n: int = 100) -> Case:
    return tet4_case(n, SEED_BASE + 2, 1.0, None, 0.3, "c2")


def config3(n: int = 40) -> Case:
    """Quadratic tets, twist 0.5 rad per unit z about x = y = 0.5, + U(+-0.01)."""
    X4, tets = kuhn_grid(n)
    X, conn = expand_quadratic(tets, X4)
    rng = np.random.default_rng(SEED_BASE + 3)
    th = 0.5 * X[:, 2]
    c, s = np.cos(th), np.sin(th)
    dx, dy = X[:, 0] - 0.5, X[:, 1] - 0.5
    x = np.stack([0.5 + c * dx - s * dy, 0.5 + s * dx + c * dy, X[:, 2]], 1)
    x += rng.uniform(-0.01, 0.01, size=x.shape)
    mu, lam = lame_from_young_poisson(NH_YOUNG, NH_POISSON)
    return Case("c3", "tet10", x, X, conn, {"mu": mu, "lambda": lam})


def config4(N: int = 1000) -> Case:
    """StVK membrane + hinge bending cloth (scenes/cloth_drop.json material)."""
    X, tris, h = cloth_grid(N)
    rng = np.random.default_rng(SEED_BASE + 4)
    x = X.copy()
    x[:, 2] += rng.normal(0.0, 0.01 * h, size=X.shape[0])
    mu, lam = lame_from_young_poisson(1e4, 0.3)
    dmi, area = cloth_rest_frames(X, tris)
    flaps = interior_edge_flaps(tris)
    return Case("c4", "cloth", x, X, tris, {"mu": mu, "lambda": lam, "kb": 1e-4},
                {"dm2inv": dmi, "area": area, "flaps": flaps})


def config5(n: int = 100, n_pairs: int = 4_000_000) -> Case:
    """Config-2 tets + inertia (dt = 1/60, rho = 1) + point-triangle barrier pairs."""
    base = tet4_case(n, SEED_BASE + 5, 1.0, None, 0.3, "c5")
    rng = np.random.default_rng(SEED_BASE + 50)
    d_hat = 1e-3
    pairs, off, _ = point_triangle_pairs(rng, base.x, n_pairs, 1.0 / n, d_hat)
    mass = lumped_mass(base.X, base.conn, 1.0)
    extra = {"pairs": pairs, "offsets": off, "mass": mass, "x_prev": base.X.copy(),
             "v": np.zeros_like(base.X)}
    params = dict(base.params)
    params.update({"dt": 1.0 / 60.0, "kappa": 1e4, "dhat": d_hat})
    return Case("c5", "contact", base.x, base.X, base.conn, params, extra)


def bending_Q_for(case: Case) -> np.ndarray:
    return bending_Q(case.X, case.extra["flaps"])
