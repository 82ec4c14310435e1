"""Problem descriptions of the BASELINE.json configurations (2D, the element
family the reference implements: dQ1-SIPG displacement, RT0-type face flux,
dQ0 pressure) and of the reference's recorded Terzaghi
run. A ProblemSpec feeds both the device assembly (pdg_ops_assemble) and the
CPU oracle (tests only)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

TAGS = ("left", "right", "bottom", "top")
TAGS3 = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")  # 3D extension
DISP = {"fixed": 0, "traction": 1, "roller_x": 2, "roller_y": 3, "roller_z": 4}
FLOW = {"pressure": 0, "no_flow": 1}

K_SEED = 1801  # per-cell permeability field (config 1, config 3)
LAYER_SEED = 1804  # layered permeability (config 2)
X_SEED = 4984  # SpMV input vector (config 3)


def lame_from_young(E: float, nu: float):
    """Plane-strain Lame parameters (the reference takes lambda, mu directly,
    problems.hpp:15-26)."""
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


@dataclass
class ProblemSpec:
    nx: int
    ny: int
    lx: float = 1.0
    ly: float = 1.0
    lam: float = 1.0
    mu: float = 1.0
    k_perm: float = 1.0
    eta: float = 1.0
    biot_m: float = 10.0
    biot_b: float = 0.8
    penalty: float = 10.0
    k_perm_cells: np.ndarray | None = None
    disp: dict = field(default_factory=dict)  # tag -> (kind, (d0, d1))
    flow: dict = field(default_factory=dict)  # tag -> (kind, value)

    def to_dict(self):
        return dict(nx=self.nx, ny=self.ny, lx=self.lx, ly=self.ly, lam=self.lam, mu=self.mu, k_perm=self.k_perm,
                    eta=self.eta, biot_m=self.biot_m, biot_b=self.biot_b, penalty=self.penalty,
                    k_perm_cells=self.k_perm_cells, disp=self.disp, flow=self.flow)

    def to_struct(self):
        p = _lib.Problem()
        p.nx, p.ny, p.lx, p.ly = self.nx, self.ny, self.lx, self.ly
        p.lam, p.mu, p.k_perm, p.eta = self.lam, self.mu, self.k_perm, self.eta
        p.biot_m, p.biot_b, p.penalty = self.biot_m, self.biot_b, self.penalty
        keep = None
        if self.k_perm_cells is not None:
            keep = np.ascontiguousarray(self.k_perm_cells, dtype=np.float64)
            assert keep.size == self.nx * self.ny
            p.k_perm_cells = keep.ctypes.data_as(C.POINTER(C.c_double))
        for s, tag in enumerate(TAGS):
            kind, data = self.disp[tag]
            p.disp_kind[s] = DISP[kind]
            p.disp_data[s][0], p.disp_data[s][1] = data
            fk, fv = self.flow[tag]
            p.flow_kind[s] = FLOW[fk]
            p.flow_data[s] = fv
        return p, keep

    @property
    def n_cells(self):
        return self.nx * self.ny

    @property
    def sizes(self):
        n = self.nx * self.ny
        n_q = self.nx * (self.ny + 1) + (self.nx + 1) * self.ny
        return 8 * n, n_q, n


@dataclass
class ProblemSpec3:
    """3D extension (BASELINE configs 2 and 4; no reference counterpart, the reference is 2D
    only): nx x ny x nz hexahedra, cell c = (k ny + j) nx + i, boundary tags TAGS3."""
    nx: int
    ny: int
    nz: int
    lx: float = 1.0
    ly: float = 1.0
    lz: float = 1.0
    lam: float = 1.0
    mu: float = 1.0
    k_perm: float = 1.0
    eta: float = 1.0
    biot_m: float = 10.0
    biot_b: float = 0.8
    penalty: float = 10.0
    k_perm_cells: np.ndarray | None = None
    disp: dict = field(default_factory=dict)  # tag -> (kind, (d0, d1, d2))
    flow: dict = field(default_factory=dict)  # tag -> (kind, value)

    def to_dict(self):
        return dict(nx=self.nx, ny=self.ny, nz=self.nz, lx=self.lx, ly=self.ly, lz=self.lz, lam=self.lam,
                    mu=self.mu, k_perm=self.k_perm, eta=self.eta, biot_m=self.biot_m, biot_b=self.biot_b,
                    penalty=self.penalty, k_perm_cells=self.k_perm_cells, disp=self.disp, flow=self.flow)

    def to_struct(self):
        p = _lib.Problem3()
        p.nx, p.ny, p.nz, p.lx, p.ly, p.lz = self.nx, self.ny, self.nz, self.lx, self.ly, self.lz
        p.lam, p.mu, p.k_perm, p.eta = self.lam, self.mu, self.k_perm, self.eta
        p.biot_m, p.biot_b, p.penalty = self.biot_m, self.biot_b, self.penalty
        keep = None
        if self.k_perm_cells is not None:
            keep = np.ascontiguousarray(self.k_perm_cells, dtype=np.float64)
            assert keep.size == self.nx * self.ny * self.nz
            p.k_perm_cells = keep.ctypes.data_as(C.POINTER(C.c_double))
        for s, tag in enumerate(TAGS3):
            kind, data = self.disp[tag]
            p.disp_kind[s] = DISP[kind]
            for k in range(3):
                p.disp_data[s][k] = data[k]
            fk, fv = self.flow[tag]
            p.flow_kind[s] = FLOW[fk]
            p.flow_data[s] = fv
        return p, keep

    @property
    def n_cells(self):
        return self.nx * self.ny * self.nz

    @property
    def sizes(self):
        n = self.n_cells
        n_q = self.nx * self.ny * (self.nz + 1) + self.nx * (self.ny + 1) * self.nz + (self.nx + 1) * self.ny * self.nz
        return 24 * n, n_q, n


def lognormal_field(seed: int, n: int, sigma: float = 1.0) -> np.ndarray:
    """K_c = exp(sigma z_c), z ~ N(0,1) i.i.d. (mt19937_64 + Box-Muller,
    DESIGN.md); generated by the library's host utility."""
    out = np.empty(n, dtype=np.float64)
    _lib.lib().pdg_util_lognormal(seed, n, sigma, out.ctypes.data_as(_lib.DP))
    return out


def uniform_vector(seed: int, n: int) -> np.ndarray:
    """x_i = -1 + 2 ((mt19937_64 >> 11) 2^-53)."""
    out = np.empty(n, dtype=np.float64)
    _lib.lib().pdg_util_uniform(seed, n, out.ctypes.data_as(_lib.DP))
    return out


def baseline_material():
    """BASELINE config 0 material: E = 1e4, nu = 0.3, b = 0.9, M = 1e3, eta = 1, K = 1."""
    lam, mu = lame_from_young(1e4, 0.3)
    return dict(lam=lam, mu=mu, k_perm=1.0, eta=1.0, biot_m=1e3, biot_b=0.9)


def baseline_bcs():
    """u = 0 bottom, traction (0,-1) top, traction-free left/right; p = 0 top,
    no-flux elsewhere (BASELINE config 0)."""
    disp = {"left": ("traction", (0.0, 0.0)), "right": ("traction", (0.0, 0.0)),
            "bottom": ("fixed", (0.0, 0.0)), "top": ("traction", (0.0, -1.0))}
    flow = {"left": ("no_flow", 0.0), "right": ("no_flow", 0.0), "bottom": ("no_flow", 0.0),
            "top": ("pressure", 0.0)}
    return disp, flow


def config0() -> ProblemSpec:
    disp, flow = baseline_bcs()
    return ProblemSpec(nx=16, ny=16, disp=disp, flow=flow, **baseline_material())


def config1(n: int = 128, seed: int = K_SEED) -> ProblemSpec:
    disp, flow = baseline_bcs()
    return ProblemSpec(nx=n, ny=n, disp=disp, flow=flow, k_perm_cells=lognormal_field(seed, n * n),
                       **baseline_material())


def config3(n: int) -> ProblemSpec:
    """SpMV sweep operator: config-1 element pair, material and K recipe at n x n."""
    return config1(n)


def layered_permeability(n_layers: int, nx: int, ny: int, nz: int, seed: int = LAYER_SEED) -> np.ndarray:
    """Config 2: n_layers horizontal layers, log10 K ~ U(-3, 0) per layer from the seed
    (u = (x + 1) / 2 with x the library's seeded uniform in (-1, 1)); cell layer = k n_layers // nz."""
    u = 0.5 * (uniform_vector(seed, n_layers) + 1.0)
    k_layer = 10.0 ** (-3.0 + 3.0 * u)
    layer = (np.arange(nz) * n_layers) // nz
    return np.repeat(k_layer[layer], nx * ny)


def config2(n: int = 32, seed: int = LAYER_SEED) -> ProblemSpec3:
    """BASELINE config 2 (3D extension): unit cube, n^3 hexahedra, config-0 material (3D Lame
    parameters from E, nu), 8 permeability layers; u = 0 on the bottom (zlo), traction (0,0,-1) on
    the top, traction-free sides; p = 0 on the top, no flux elsewhere."""
    free = ("traction", (0.0, 0.0, 0.0))
    disp = {"xlo": free, "xhi": free, "ylo": free, "yhi": free, "zlo": ("fixed", (0.0, 0.0, 0.0)),
            "zhi": ("traction", (0.0, 0.0, -1.0))}
    flow = {t: ("no_flow", 0.0) for t in TAGS3}
    flow["zhi"] = ("pressure", 0.0)
    return ProblemSpec3(nx=n, ny=n, nz=n, disp=disp, flow=flow, k_perm_cells=layered_permeability(8, n, n, n, seed),
                        **baseline_material())


def config4(n: int = 96, seed: int = K_SEED) -> ProblemSpec3:
    """BASELINE config 4 (3D extension): n^3 hexahedra, i.i.d. per-cell lognormal permeability
    (sigma = 1.5) from the seed, dG(1), 8 slabs; boundary data as config 2. The full size (96^3)
    is out of reach of the reference's exact preconditioner; the bench
    runs it at a reduced n."""
    spec = config2(n)
    spec.k_perm_cells = lognormal_field(seed, n * n * n, 1.5)
    return spec


def terzaghi_recorded() -> ProblemSpec:
    """The reference's recorded run proj/out/iterations.csv: Terzaghi column,
    1 x 8 square cells, desk material (lambda = mu = 1, M = 10, b = 0.8)."""
    disp = {"left": ("roller_x", (0.0, 0.0)), "right": ("roller_x", (0.0, 0.0)),
            "bottom": ("roller_y", (0.0, 0.0)), "top": ("traction", (0.0, -1.0))}
    flow = {"left": ("no_flow", 0.0), "right": ("no_flow", 0.0), "bottom": ("no_flow", 0.0),
            "top": ("pressure", 0.0)}
    return ProblemSpec(nx=1, ny=8, lx=1.0 / 8.0, ly=1.0, disp=disp, flow=flow)


# Run settings of the configurations (r, T, slabs, GMRES restart, tol).
RUNS = {
    "config0": dict(r=0, T=1.0, n_slabs=10, restart=50, tol=1e-10),
    "config1": dict(r=1, T=1.0, n_slabs=20, restart=50, tol=1e-10),
    "config2": dict(r=0, T=1.0, n_slabs=10, restart=50, tol=1e-10),
    "config4": dict(r=1, T=1.0, n_slabs=8, restart=50, tol=1e-10),
    "terzaghi_recorded": dict(r=0, T=0.2, n_slabs=10, restart=100, tol=1e-8),
}
