"""Problem description with the reference API (discretization.py:38-102, 187-218).

Only the setup data lives here: the wavenumber / geometry / incident wave,
the impedance coefficient, the owning subdomain of the scatterer and its
staircase cells.  The factorisation and every solve run on the GPU
(interface_system.GpuInterfaceSystem -> libhsb200).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .indexing import MultiIndex, Partition

FACES = ("west", "east", "south", "north")  # discretization.py:30
COMPACT_FACE_ORDER = ("west", "south", "north", "east")  # m-order of one owner's blocks
MONO_GUARD = 250_000


@dataclass(frozen=True)
class Scatterer:
    center: tuple[float, float] = (0.0, 0.0)
    radius: float = 1.0


@dataclass(frozen=True)
class ProblemSpec:
    """discretization.py:46-83 (same fields, defaults and validation)."""

    kappa: float
    cells_per_side: int
    subdomain_side: float = 2.5
    scatterer: Scatterer | None = field(default_factory=Scatterer)
    incident_direction: tuple[float, float] = (1.0, 0.0)

    def __post_init__(self):
        if self.kappa <= 0:
            raise ValueError(f"kappa must be positive, got {self.kappa}")
        if self.subdomain_side <= 0:
            raise ValueError(f"subdomain_side must be positive, got {self.subdomain_side}")
        if self.cells_per_side < 4:
            raise ValueError(f"cells_per_side must be >= 4, got {self.cells_per_side}")
        if self.incident_direction[0] == 0 and self.incident_direction[1] == 0:
            raise ValueError("incident_direction must be nonzero")

    @property
    def h(self) -> float:
        return self.subdomain_side / self.cells_per_side

    @property
    def origin(self) -> tuple[float, float]:
        return (-self.subdomain_side / 2.0, -self.subdomain_side / 2.0)

    def incident_wave(self, x, y, direction=None):
        return plane_wave(self.kappa, self.incident_direction if direction is None else direction, x, y)


@dataclass(frozen=True)
class ImpedanceSpec:
    """discretization.py:86-102: tau, nonzero imaginary part required."""

    coefficient: complex

    def __post_init__(self):
        if complex(self.coefficient).imag == 0:
            raise ValueError("impedance coefficient must have nonzero imaginary part")

    @classmethod
    def for_problem(cls, spec) -> "ImpedanceSpec":
        return cls(1j * spec.kappa)


def cell_centres(spec, i):
    """Cell centres of subdomain i as (x, y) grids [iy, ix] (discretization.py:143-149)."""
    n, h, side = spec.cells_per_side, spec.h, spec.subdomain_side
    ox, oy = spec.origin
    xs = ox + (i[0] - 1) * side + (np.arange(n) + 0.5) * h
    ys = oy + (i[1] - 1) * side + (np.arange(n) + 0.5) * h
    return np.meshgrid(xs, ys)


def scatterer_subdomain(spec, partition) -> MultiIndex | None:
    """Subdomain whose open interior strictly contains the disk (discretization.py:203-218)."""
    sc = spec.scatterer
    if sc is None:
        return None
    cx, cy = sc.center
    r = sc.radius
    ox, oy = spec.origin
    side = spec.subdomain_side
    for i in partition.subdomains:
        x0, y0 = ox + (i[0] - 1) * side, oy + (i[1] - 1) * side
        if x0 < cx - r and cx + r < x0 + side and y0 < cy - r and cy + r < y0 + side:
            return MultiIndex(*i)
    raise ValueError("scatterer must lie strictly inside one subdomain, away from interfaces")


def scatterer_cells(spec, partition, i=None) -> tuple[MultiIndex | None, np.ndarray]:
    """(home subdomain, staircase cells of the disk) (discretization.py:187-200)."""
    home = scatterer_subdomain(spec, partition)
    if home is None or (i is not None and MultiIndex(*i) != home):
        return home, np.empty(0, dtype=np.intp)
    X, Y = cell_centres(spec, home)
    cx, cy = spec.scatterer.center
    cells = np.flatnonzero(((X - cx) ** 2 + (Y - cy) ** 2 < spec.scatterer.radius ** 2).ravel())
    if cells.size == 0:
        raise ValueError(f"cells_per_side={spec.cells_per_side} too coarse: no cell center inside the scatterer")
    return home, cells


def lifting_data(spec, partition, directions=None) -> tuple[MultiIndex | None, np.ndarray]:
    """Dirichlet data -u_inc on the scatterer cells (discretization.py:326-328) for
    one or several incident directions: array [ncells, nrhs] complex."""
    home, cells = scatterer_cells(spec, partition)
    if home is None:
        return None, np.zeros((0, 1), dtype=complex)
    X, Y = cell_centres(spec, home)
    x, y = X.ravel()[cells], Y.ravel()[cells]
    if directions is None:
        # the spec's own incident_wave (discretization.py:79-83): also a reference ProblemSpec's
        return home, -np.asarray(spec.incident_wave(x, y))[:, None]
    return home, np.stack([-plane_wave(spec.kappa, d, x, y) for d in directions], axis=1)


def plane_wave(kappa, direction, x, y):
    """exp(i kappa d.x / |d|) (discretization.py:79-83) for any direction d."""
    dx, dy = direction
    return np.exp(1j * kappa * (dx * x + dy * y) / np.hypot(dx, dy))


def face_cells(n: int) -> dict[str, np.ndarray]:
    """Boundary cells per face, increasing global coordinate (discretization.py:151-158)."""
    idx = np.arange(n * n).reshape(n, n)
    return {"west": idx[:, 0].copy(), "east": idx[:, -1].copy(), "south": idx[0, :].copy(), "north": idx[-1, :].copy()}


@dataclass
class SubdomainInfo:
    """What remains of LocalOperator (discretization.py:116-184) on the host:
    ghost coefficients, faces and scatterer cells.  The factorisation itself
    lives on the GPU (`GpuInterfaceSystem.schur_map(i)`)."""

    subdomain: MultiIndex
    n: int
    h: float
    tau: complex
    ghost_d: complex
    ghost_s: complex
    rhs_coeff: complex
    faces: dict
    interface_faces: dict
    dirichlet_cells: np.ndarray

    @classmethod
    def build(cls, spec, imp, partition: Partition, i) -> "SubdomainInfo":
        i = MultiIndex(*i)
        n, h = spec.cells_per_side, spec.h
        tau = complex(imp.coefficient)
        d, s = 1.0 / h - tau / 2.0, 1.0 / h + tau / 2.0
        steps = {"west": (-1, 0), "east": (1, 0), "south": (0, -1), "north": (0, 1)}
        iface = {}
        for f, (a, b) in steps.items():
            j = MultiIndex(i.i1 + a, i.i2 + b)
            if 1 <= j.i1 <= partition.n1 and 1 <= j.i2 <= partition.n2:
                iface[f] = j
        _, cells = scatterer_cells(spec, partition, i)
        return cls(i, n, h, tau, d, s, 1.0 / (h * h * d), face_cells(n), iface, cells)

    def face_toward(self, j) -> str:
        for f, nb in self.interface_faces.items():
            if nb == MultiIndex(*j):
                return f
        raise ValueError(f"{tuple(j)} is not a neighbor of {tuple(self.subdomain)}")
