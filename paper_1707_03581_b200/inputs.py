"""Seeded synthetic inputs: Kuhn-split box meshes and the BASELINE.json configurations.

This module is shared by the CUDA path (via ``bench.py`` / the tests) and by the CPU
oracle tests.  It holds NONE of the method's arithmetic: it only produces the input
arrays that go through ``thermo_create_mesh`` (node coordinates, tetrahedra, tagged
boundary triangles) and the scalar parameters of each configuration.

Paper context (PAPER.md = /root/reference/PAPER.md, cited as P:line):
  * two independently meshed domains, fixed stand/rail and moving stock
  * the stock slides along the rail, s(t) = a sin(2 pi t / eps) + s0
  * Robin boundaries i = 1 (environment), 2 (cooling), 3 (floor)
  * T_env = 24 C at the floor rising 0.5 C over 2 m
The paper's CAD geometry (Naumann2016) is not available; the synthetic boxes
below stand in for it.

Mesh recipe: every lattice cell of a union of axis-aligned boxes is split
into 6 Kuhn tetrahedra along its (0,0,0)-(1,1,1) diagonal, the same way in every cell,
so the mesh is conforming.  Nodes are numbered in lattice order (x fastest, then y,
then z).  Optional jitter moves every node by U(-j h, j h) per coordinate, drawn from a
splitmix64 hash of (seed, lattice node index, axis), except along any axis normal to a
boundary face the node lies on -- this keeps every boundary face planar (so the
interface plane stays a plane) and the total volume exact.

Boundary-face tags used by all configs:
  0 = insulated, 1 = environment Robin, 2 = cooling Robin, 3 = floor Robin,
  4 = interface (rail top on the fixed part, stock bottom on the moving part).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

TAG_INSULATED = 0
TAG_ENV = 1
TAG_COOL = 2
TAG_FLOOR = 3
TAG_IFACE = 4

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)).astype(np.uint64)
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, index: np.ndarray, stream: int) -> np.ndarray:
    """U[0,1) from splitmix64 of (seed, index, stream); top 53 bits."""
    key = (np.uint64(seed) << np.uint64(40)) ^ (index.astype(np.uint64) * np.uint64(8) + np.uint64(stream))
    return (splitmix64(key) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


@dataclasses.dataclass
class Mesh:
    """Input arrays of one part, exactly as passed to thermo_create_mesh."""
    xyz: np.ndarray        # float64 [n_nodes, 3]
    tets: np.ndarray       # int32 [n_tets, 4], positive orientation
    bfaces: np.ndarray     # int32 [n_bfaces, 3], outward orientation
    bface_tag: np.ndarray  # int32 [n_bfaces]

    @property
    def n_nodes(self) -> int:
        return int(self.xyz.shape[0])

    @property
    def n_tets(self) -> int:
        return int(self.tets.shape[0])


# Kuhn permutations: (first, second, third) axis of the monotone path 000 -> 111.
_PERMS = [(0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2)]
_PERM_EVEN = [True, True, True, False, False, False]


def kuhn_box_union(origin: Sequence[float], h: Sequence[float], shape: Sequence[int],
                   boxes: Sequence[Tuple[int, int, int, int, int, int]],
                   tag_fn: Callable[[int, int, np.ndarray], np.ndarray],
                   jitter: float = 0.0, seed: int = 0) -> Mesh:
    """Kuhn-split tetrahedral mesh of a union of lattice boxes.

    origin, h: lattice origin and spacing per axis; shape = (nx, ny, nz) cells of the
    bounding lattice; boxes = cell-index ranges (i0, i1, j0, j1, k0, k1), half-open.
    tag_fn(axis, side, centers[n,3]) -> int32 tags of boundary faces.
    """
    nx, ny, nz = (int(s) for s in shape)
    h = np.asarray(h, dtype=np.float64)
    origin = np.asarray(origin, dtype=np.float64)
    cell = np.zeros((nz, ny, nx), dtype=bool)
    for (i0, i1, j0, j1, k0, k1) in boxes:
        cell[k0:k1, j0:j1, i0:i1] = True
    # active nodes: any adjacent cell active
    pad = np.zeros((nz + 2, ny + 2, nx + 2), dtype=bool)
    pad[1:-1, 1:-1, 1:-1] = cell
    node = np.zeros((nz + 1, ny + 1, nx + 1), dtype=bool)
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                node |= pad[dz:dz + nz + 1, dy:dy + ny + 1, dx:dx + nx + 1]
    flat = node.ravel()
    nid = np.full(flat.shape, -1, dtype=np.int64)
    nid[flat] = np.arange(int(flat.sum()), dtype=np.int64)
    nid = nid.reshape(node.shape)
    gidx = np.nonzero(flat)[0]                       # global lattice index of each node
    kk, jj, ii = np.unravel_index(gidx, node.shape)
    lat = np.stack([ii, jj, kk], axis=1).astype(np.float64)

    # tetrahedra
    ck, cj, ci = np.nonzero(cell)

    def corner(dx, dy, dz):
        return nid[ck + dz, cj + dy, ci + dx]

    c000 = corner(0, 0, 0)
    c111 = corner(1, 1, 1)
    tets = []
    for perm, even in zip(_PERMS, _PERM_EVEN):
        off1 = [0, 0, 0]
        off1[perm[0]] = 1
        off2 = list(off1)
        off2[perm[1]] = 1
        v1 = corner(*off1)
        v2 = corner(*off2)
        if even:
            tets.append(np.stack([c000, v1, v2, c111], axis=1))
        else:
            tets.append(np.stack([c000, v2, v1, c111], axis=1))
    tets = np.stack(tets, axis=1).reshape(-1, 4).astype(np.int32)

    # boundary faces: active cell whose neighbour across the face is inactive
    faces, tags, fixed_axis_nodes = [], [], [[], [], []]
    for axis in range(3):
        u, v = [a for a in range(3) if a != axis]
        for side in (0, 1):
            step = [0, 0, 0]
            step[axis] = 1 if side == 1 else -1
            # neighbour activity via the padded array
            nb = pad[1 + step[2]:1 + step[2] + nz, 1 + step[1]:1 + step[1] + ny,
                     1 + step[0]:1 + step[0] + nx]
            bk, bj, bi = np.nonzero(cell & ~nb)
            if bk.size == 0:
                continue

            def fc(du, dv):
                off = [0, 0, 0]
                off[axis] = side
                off[u] += du
                off[v] += dv
                return nid[bk + off[2], bj + off[1], bi + off[0]]

            a00, a10, a11, a01 = fc(0, 0), fc(1, 0), fc(1, 1), fc(0, 1)
            # (u, v, axis) right-handed for axis 0 and 2, left-handed for axis 1
            outward_is_uv = (side == 1) if axis != 1 else (side == 0)
            if outward_is_uv:
                t1 = np.stack([a00, a10, a11], axis=1)
                t2 = np.stack([a00, a11, a01], axis=1)
            else:
                t1 = np.stack([a00, a11, a10], axis=1)
                t2 = np.stack([a00, a01, a11], axis=1)
            f = np.stack([t1, t2], axis=1).reshape(-1, 3)
            centers = np.zeros((bk.size, 3))
            centers[:, 0] = bi + 0.5
            centers[:, 1] = bj + 0.5
            centers[:, 2] = bk + 0.5
            centers[:, axis] = (np.array([bi, bj, bk])[axis] + side)
            centers = origin + centers * h
            tg = np.asarray(tag_fn(axis, side, centers), dtype=np.int32)
            faces.append(f)
            tags.append(np.repeat(tg, 2))
            fixed_axis_nodes[axis].append(np.concatenate([a00, a10, a11, a01]))
    bfaces = np.concatenate(faces).astype(np.int32)
    bface_tag = np.concatenate(tags).astype(np.int32)

    xyz = origin + lat * h
    if jitter > 0.0:
        n = xyz.shape[0]
        for axis in range(3):
            free = np.ones(n, dtype=bool)
            if fixed_axis_nodes[axis]:
                free[np.unique(np.concatenate(fixed_axis_nodes[axis]))] = False
            r = uniform01(seed, gidx, axis)
            xyz[:, axis] += np.where(free, (2.0 * r - 1.0) * jitter * h[axis], 0.0)
    return Mesh(xyz=np.ascontiguousarray(xyz), tets=np.ascontiguousarray(tets),
                bfaces=np.ascontiguousarray(bfaces), bface_tag=np.ascontiguousarray(bface_tag))


@dataclasses.dataclass
class Scenario:
    """Motion s(t) = s0 + amp sin(2 pi t / period) along dir and friction
    heat eta(t) = eta0 (1 + eta_amp sin(2 pi t / eta_period))."""
    s0: float
    amp: float
    period: float
    eta0: float
    eta_amp: float = 0.0
    eta_period: float = 1.0
    dir: Tuple[float, float, float] = (1.0, 0.0, 0.0)


@dataclasses.dataclass
class Robin:
    """Robin data of one (part, tag): alpha_i and T_i(x) = T_ref + grad . x."""
    part: int
    tag: int
    alpha: float
    T_ref: float
    grad: Tuple[float, float, float] = (0.0, 0.0, 0.0)


@dataclasses.dataclass
class Config:
    name: str
    fixed: Mesh
    moving: Mesh
    nu: float
    rho_cp: float
    alpha_iface: float
    robin: List[Robin]
    scenarios: List[Scenario]
    T0: float
    dt: float
    nsteps: int
    iface_tag: int = TAG_IFACE
    description: str = ""

    @property
    def n_dof(self) -> int:
        return self.fixed.n_nodes + self.moving.n_nodes

    @property
    def n_scen(self) -> int:
        return len(self.scenarios)


# ---------------------------------------------------------------------------------
# Tag rules
# ---------------------------------------------------------------------------------

def _rail_box_tags(axis, side, centers):
    """Fixed rail box: floor at z=0 (tag 3), rail top = interface (tag 4), others env."""
    t = np.full(centers.shape[0], TAG_ENV, dtype=np.int32)
    if axis == 2 and side == 0:
        t[:] = TAG_FLOOR
    if axis == 2 and side == 1:
        t[:] = TAG_IFACE
    return t


def _stock_tags(axis, side, centers):
    """Moving stock: bottom = interface (tag 4), +y back face = cooling (tag 2), others env.
    Reading DESIGN.md R9: "back of the stock" (P:5) is the +y face."""
    t = np.full(centers.shape[0], TAG_ENV, dtype=np.int32)
    if axis == 2 and side == 0:
        t[:] = TAG_IFACE
    if axis == 1 and side == 1:
        t[:] = TAG_COOL
    return t


def _make_lshape_tags(rail_x, rail_y, rail_top_z, tol):
    def fn(axis, side, centers):
        t = np.full(centers.shape[0], TAG_ENV, dtype=np.int32)
        if axis == 2 and side == 0:
            t[np.abs(centers[:, 2]) < tol] = TAG_FLOOR
        if axis == 2 and side == 1:
            on = ((np.abs(centers[:, 2] - rail_top_z) < tol)
                  & (centers[:, 0] > rail_x[0]) & (centers[:, 0] < rail_x[1])
                  & (centers[:, 1] > rail_y[0]) & (centers[:, 1] < rail_y[1]))
            t[on] = TAG_IFACE
        return t
    return fn


# ---------------------------------------------------------------------------------
# Configurations (BASELINE.json configs[0..4])
# ---------------------------------------------------------------------------------

NU = 50.0            # W/mK            (BJ cfg 0)
RHO_CP = 3.6e6       # J/m^3K          (BJ cfg 0)
ALPHA_IFACE = 1000.  # W/m^2K          (BJ cfg 0)


def _std_robin():
    """BJ cfg 0: alpha1=10, T1=24+0.25 z on other faces; alpha3=50, T3=24 on the rail
    bottom; alpha2=200, T2=18 on the stock back face.  T1 rises 0.5 C over 2 m."""
    r = []
    for part in (0, 1):
        r.append(Robin(part, TAG_ENV, 10.0, 24.0, (0.0, 0.0, 0.25)))
    r.append(Robin(0, TAG_FLOOR, 50.0, 24.0))
    r.append(Robin(1, TAG_COOL, 200.0, 18.0))
    return r


def rail_pair(rail_cells, stock_cells, jitter=0.0, seed=1707):
    """cfg 0/1 geometry: rail [0,1]x[0,0.2]x[0,0.1], stock 0.25x0.2x0.1 at z in [0.1,0.2]
    (reference frame x in [0, 0.25])."""
    rx, ry, rz = rail_cells
    sx, sy, sz = stock_cells
    fixed = kuhn_box_union((0.0, 0.0, 0.0), (1.0 / rx, 0.2 / ry, 0.1 / rz), (rx, ry, rz),
                           [(0, rx, 0, ry, 0, rz)], _rail_box_tags, jitter, seed)
    moving = kuhn_box_union((0.0, 0.0, 0.1), (0.25 / sx, 0.2 / sy, 0.1 / sz), (sx, sy, sz),
                            [(0, sx, 0, sy, 0, sz)], _stock_tags, jitter, seed + 1)
    return fixed, moving


def lshape_pair(h_fixed, h_stock, jitter=0.1, seed=1707):
    """cfg 2/3 geometry: column [0,.6]x[0,.6]x[0,2], foot [.6,2.1]x[0,.6]x[0,.25],
    rail [.6,2.1]x[.2,.4]x[.25,.35]; stock 0.4x0.2x0.2 at y in [.2,.4], z in [.35,.55]."""
    def c(v, h):
        return int(round(v / h))
    hf = h_fixed
    boxes = [(0, c(0.6, hf), 0, c(0.6, hf), 0, c(2.0, hf)),
             (c(0.6, hf), c(2.1, hf), 0, c(0.6, hf), 0, c(0.25, hf)),
             (c(0.6, hf), c(2.1, hf), c(0.2, hf), c(0.4, hf), c(0.25, hf), c(0.35, hf))]
    shape = (c(2.1, hf), c(0.6, hf), c(2.0, hf))
    tagf = _make_lshape_tags((0.6, 2.1), (0.2, 0.4), 0.35, 0.25 * hf)
    fixed = kuhn_box_union((0.0, 0.0, 0.0), (hf, hf, hf), shape, boxes, tagf, jitter, seed)
    hs = h_stock
    sx, sy, sz = c(0.4, hs), c(0.2, hs), c(0.2, hs)
    moving = kuhn_box_union((0.0, 0.2, 0.35), (hs, hs, hs), (sx, sy, sz),
                            [(0, sx, 0, sy, 0, sz)], _stock_tags, jitter, seed + 1)
    return fixed, moving


def make_config(name: str, n_scen: Optional[int] = None, jitter: Optional[float] = None) -> Config:
    """Build one named configuration.

    cfg0..cfg4 are BASELINE.json configs[0..4]; "small" and "medium" are extra parity
    sizes (same geometry as cfg 0/1, several SELL slices + a ragged tail); "paper" has the DoF
    count of the paper's machine model (16,626 DoF; here 16,870) on the same geometry, for
    the look-ahead measurements.  `jitter` overrides the configuration's node jitter (fraction
    of h)."""
    if name in ("cfg0", "small", "medium", "paper", "cfg1", "cfg4"):
        cells = {"cfg0": ((16, 4, 2), (5, 3, 2)),
                 "small": ((32, 8, 4), (10, 6, 3)),
                 "medium": ((64, 16, 8), (20, 12, 6)),
                 "paper": ((72, 18, 9), (24, 14, 7)),
                 "cfg1": ((128, 32, 16), (40, 24, 12)),
                 "cfg4": ((128, 32, 16), (40, 24, 12))}[name]
        fixed, moving = rail_pair(*cells, jitter=0.0 if jitter is None else jitter)
        if name == "cfg4":
            S = 64 if n_scen is None else n_scen
            scen = [Scenario(0.375, 0.375, 20.0 + k, 100.0 + 15.0 * k) for k in range(S)]
            dt, nsteps = 1.0, 500
        elif name == "cfg0":
            scen = [Scenario(0.375, 0.375, 60.0, 500.0)]
            dt, nsteps = 1.0, 100
        elif name == "cfg1":
            scen = [Scenario(0.375, 0.375, 60.0, 500.0, 0.5, 20.0)]
            dt, nsteps = 0.5, 1000
        else:
            scen = [Scenario(0.375, 0.375, 60.0, 500.0, 0.5, 20.0)]
            dt, nsteps = 0.5, {"small": 50, "medium": 30, "paper": 30}[name]
        return Config(name, fixed, moving, NU, RHO_CP, ALPHA_IFACE, _std_robin(), scen,
                      24.0, dt, nsteps, description=f"rail pair {cells}")
    if name in ("cfg2", "cfg3"):
        hf, hs, nsteps = {"cfg2": (0.01, 0.004, 3600), "cfg3": (0.005, 0.002, 200)}[name]
        fixed, moving = lshape_pair(hf, hs, jitter=0.1 if jitter is None else jitter)
        scen = [Scenario(1.15, 0.5, 30.0, 500.0)]
        return Config(name, fixed, moving, NU, RHO_CP, ALPHA_IFACE, _std_robin(), scen,
                      24.0, 1.0, nsteps, description=f"L-shape stand h={hf}, stock h={hs}")
    raise ValueError(f"unknown config {name!r}")


def two_slab_pair(rail_cells=(6, 4, 2), stock_cells=(5, 3, 4), jitter=0.0, seed=7):
    """Laterally homogeneous two-slab pair with equal 0.3x0.2 footprints and non-matching
    lattices: rail 0.3x0.2x0.1, stock 0.3x0.2x0.1 on top.  Only bottom (tag 3) and top
    (tag 2) faces are Robin; the sides are insulated (tag 0); the contact is tag 4."""
    def rail_tags(axis, side, c):
        t = np.full(c.shape[0], TAG_INSULATED, dtype=np.int32)
        if axis == 2:
            t[:] = TAG_FLOOR if side == 0 else TAG_IFACE
        return t

    def stock_tags(axis, side, c):
        t = np.full(c.shape[0], TAG_INSULATED, dtype=np.int32)
        if axis == 2:
            t[:] = TAG_IFACE if side == 0 else TAG_COOL
        return t
    rx, ry, rz = rail_cells
    sx, sy, sz = stock_cells
    fixed = kuhn_box_union((0, 0, 0), (0.3 / rx, 0.2 / ry, 0.1 / rz), rail_cells,
                           [(0, rx, 0, ry, 0, rz)], rail_tags, jitter, seed)
    moving = kuhn_box_union((0, 0, 0.1), (0.3 / sx, 0.2 / sy, 0.1 / sz), stock_cells,
                            [(0, sx, 0, sy, 0, sz)], stock_tags, jitter, seed + 1)
    return fixed, moving


def scenario_scalars(scen: Scenario, t: float) -> Tuple[float, float]:
    """(s(t), eta(t)) for one scenario -- the input time law of the configs."""
    s = scen.s0 + scen.amp * math.sin(2.0 * math.pi * t / scen.period)
    eta = scen.eta0 * (1.0 + scen.eta_amp * math.sin(2.0 * math.pi * t / scen.eta_period))
    return s, eta


def initial_field(cfg: Config, seed: int = 11, amp: float = 0.5) -> np.ndarray:
    """A seeded smooth-plus-noise initial temperature [n_scen, n_dof] around T0, used by
    short-horizon parity cases that start away from the uniform state."""
    n = cfg.n_dof
    idx = np.arange(n, dtype=np.int64)
    xyz = np.concatenate([cfg.fixed.xyz, cfg.moving.xyz])
    out = np.empty((cfg.n_scen, n))
    for s in range(cfg.n_scen):
        r = uniform01(seed + 101 * s, idx, 5)
        out[s] = cfg.T0 + amp * np.sin(3.0 * xyz[:, 0] + 5.0 * xyz[:, 2] + s) + 0.1 * amp * (2 * r - 1)
    return out


def permute_mesh(mesh: Mesh, seed: int) -> Tuple[Mesh, np.ndarray]:
    """The same mesh with its nodes renumbered by a seeded random permutation (an arbitrary
    caller numbering, as a CAD mesher would produce).  Returns (mesh, old_of_new):
    node k of the result is node old_of_new[k] of the input.  Tets and faces keep their order
    and orientation."""
    n = mesh.n_nodes
    old_of_new = np.argsort(uniform01(seed, np.arange(n, dtype=np.int64), 3), kind="stable")
    new_of_old = np.empty(n, dtype=np.int64)
    new_of_old[old_of_new] = np.arange(n)
    return Mesh(xyz=np.ascontiguousarray(mesh.xyz[old_of_new]),
                tets=np.ascontiguousarray(new_of_old[mesh.tets].astype(np.int32)),
                bfaces=np.ascontiguousarray(new_of_old[mesh.bfaces].astype(np.int32)),
                bface_tag=mesh.bface_tag.copy()), old_of_new


def permute_config(cfg: Config, seed: int = 99) -> Tuple[Config, np.ndarray]:
    """cfg with both parts' nodes randomly renumbered (seeded).  Returns (cfg', old_of_new) with
    old_of_new over the coupled numbering (fixed part first): T'[k] = T[old_of_new[k]]."""
    f, pf = permute_mesh(cfg.fixed, seed)
    m, pm = permute_mesh(cfg.moving, seed + 1)
    out = dataclasses.replace(cfg, name=cfg.name + "_perm", fixed=f, moving=m)
    return out, np.concatenate([pf, pm + cfg.fixed.n_nodes])
