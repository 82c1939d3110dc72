"""Seeded synthetic inputs shared by the oracle (``oracle/``) and the CUDA path.

This module holds *problem descriptions only*: grids of finite-volume cells,
IC/BC observation sites, PDE operator coefficients, observation noise levels,
right-hand sides computed from the analytic initial conditions, prediction
grids and seeded random vectors.  It contains none of the method's arithmetic
(no kernel evaluation, no Gram assembly, no solves), so that ``oracle/`` and
``paper_2406_05020_b200/`` can both consume it without sharing code
(DESIGN.md §3 "independence").

Notation follows PAPER.md:
  * a block of observations is a *factorized scheme* (PAPER.md l.306-313,
    §4 Definition): per dimension a list of 1D sites, the block's observations
    are the Cartesian product, flattened row-major (dimension 0 = time slowest);
  * every observation of a block is the functional
    ``sum_tau c_tau  prod_i L_{site_i; alpha_tau,i}`` (Eq. 15-16,
    l.244-246) where a site is an interval [a,b] (FVM cell, the functional is
    int_a^b d^m/dx^m) or a point p (u^{(m)}(p), collocation/IC/BC functionals,
    PAPER.md l.170);
  * ``output`` selects the output of a multi-output prior (Eq. 17-19).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

POINT = 0
INTERVAL = 1


@dataclass
class Kernel1D:
    """Half-integer Matérn factor nu = q + 1/2 (Eq. 12, l.215)."""
    q: int
    lengthscale: float
    variance: float = 1.0


@dataclass
class Sites:
    """1D site list of one dimension of one block (all sites of one kind)."""
    kind: int                 # POINT or INTERVAL
    lo: np.ndarray            # interval left end, or the point location
    hi: np.ndarray            # interval right end (== lo for points)

    @property
    def n(self) -> int:
        return int(self.lo.shape[0])


@dataclass
class Term:
    """One term c * D^alpha [u_output] of the (linear) operator of a block."""
    coeff: float
    order: Tuple[int, ...]
    output: int = 0


@dataclass
class Block:
    name: str
    sites: List[Sites]
    terms: List[Term]
    noise: float              # observation noise variance Sigma_jj
    deflate: bool             # True: IC/BC block solved exactly (§4.2)
    rhs: np.ndarray           # observed values y for this block (flattened)

    @property
    def shape(self) -> Tuple[int, ...]:
        return tuple(s.n for s in self.sites)

    @property
    def size(self) -> int:
        return int(np.prod(self.shape))


@dataclass
class Problem:
    name: str
    ndim: int
    kernels: List[List[Kernel1D]]     # [output][dim]
    blocks: List[Block]
    meta: dict = field(default_factory=dict)

    @property
    def n_outputs(self) -> int:
        return len(self.kernels)

    @property
    def size(self) -> int:
        return sum(b.size for b in self.blocks)

    @property
    def offsets(self) -> List[int]:
        off = [0]
        for b in self.blocks:
            off.append(off[-1] + b.size)
        return off

    def rhs(self) -> np.ndarray:
        return np.concatenate([b.rhs for b in self.blocks]).astype(np.float64)


@dataclass
class Grid:
    """Tensor prediction grid: the Cartesian product of per-dimension points."""
    points: List[np.ndarray]
    output: int = 0

    @property
    def shape(self) -> Tuple[int, ...]:
        return tuple(len(p) for p in self.points)


def cells(n: int, lo: float = 0.0, hi: float = 1.0) -> Sites:
    """n uniform cells of [lo, hi] (FVM volumes that "disjointly span the
    entire domain")."""
    e = np.linspace(lo, hi, n + 1)
    return Sites(INTERVAL, e[:-1].copy(), e[1:].copy())


def point(p: float) -> Sites:
    return Sites(POINT, np.array([p], dtype=np.float64), np.array([p], dtype=np.float64))


def points(ps: Sequence[float]) -> Sites:
    a = np.asarray(ps, dtype=np.float64)
    return Sites(POINT, a.copy(), a.copy())


# ---------------------------------------------------------------------------
# 1D heat equation u_t = kappa u_xx on [0,1]x[0,1] (BASELINE.json configs 0, 1)
# ---------------------------------------------------------------------------

def sine_series_ic(n_modes: int, seed: int) -> np.ndarray:
    """Amplitudes A_k ~ N(0, 1/k^2), k = 1..n_modes (BASELINE.json config 1)."""
    rng = np.random.default_rng(seed)
    k = np.arange(1, n_modes + 1)
    return rng.standard_normal(n_modes) / k


def heat_analytic(amps: np.ndarray, kappa: float, t: np.ndarray, x: np.ndarray) -> np.ndarray:
    """u(t,x) = sum_k A_k exp(-kappa k^2 pi^2 t) sin(k pi x): the separation-
    of-variables solution of u_t = kappa u_xx with u(t,0)=u(t,1)=0."""
    k = np.arange(1, len(amps) + 1)
    tt = np.asarray(t, dtype=np.float64)[:, None, None]
    xx = np.asarray(x, dtype=np.float64)[None, :, None]
    return np.sum(amps * np.exp(-kappa * (k * np.pi) ** 2 * tt) * np.sin(k * np.pi * xx), axis=-1)


def heat_problem(nt: int, nx: int, *, kappa: float = 0.1, ell_t: float = 0.5, ell_x: float = 0.2,
                 q: int = 2, amps: np.ndarray | None = None, jitter: float = 1e-8,
                 pde_noise: float = 0.0, name: str | None = None) -> Problem:
    """FVM problem for u_t - kappa u_xx = 0 with IC u(0,x) = sum_k A_k sin(k pi x)
    and Dirichlet-0 BC.

    Blocks (in this order):
      IC   : t = point 0,     x = nx cells, functional  int_cell u(0,x) dx
      BC0  : t = nt cells,    x = point 0,  functional  int_cell u(t,0) dt
      BC1  : t = nt cells,    x = point 1,  functional  int_cell u(t,1) dt
      PDE  : t = nt cells,    x = nx cells, functional  int_V (u_t - kappa u_xx)
    IC/BC observation noise: ``jitter * h^2`` with h the cell width (the
    prior variance of a cell integral of a unit-variance process is ~h^2);
    DESIGN.md reading R4.
    """
    if amps is None:
        amps = np.array([1.0])
    T = cells(nt)
    X = cells(nx)
    ht, hx = 1.0 / nt, 1.0 / nx
    k = np.arange(1, len(amps) + 1)
    a, b = X.lo, X.hi
    ic = np.sum(amps[None, :] * (np.cos(k[None, :] * np.pi * a[:, None]) -
                                  np.cos(k[None, :] * np.pi * b[:, None])) / (k[None, :] * np.pi), axis=1)
    blocks = [
        Block("IC", [point(0.0), X], [Term(1.0, (0, 0))], jitter * hx * hx, True, ic),
        Block("BC0", [T, point(0.0)], [Term(1.0, (0, 0))], jitter * ht * ht, True, np.zeros(nt)),
        Block("BC1", [T, point(1.0)], [Term(1.0, (0, 0))], jitter * ht * ht, True, np.zeros(nt)),
        Block("PDE", [T, X], [Term(1.0, (1, 0)), Term(-kappa, (0, 2))], pde_noise, False,
              np.zeros(nt * nx)),
    ]
    kern = [[Kernel1D(q, ell_t, 1.0), Kernel1D(q, ell_x, 1.0)]]
    return Problem(name or f"heat1d_{nt}x{nx}", 2, kern, blocks,
                   meta=dict(kind="heat1d", kappa=kappa, amps=np.asarray(amps), nt=nt, nx=nx))


def config0() -> Problem:
    """BASELINE.json configs[0]: 16x16 cells, u0 = sin(pi x), Matérn-5/2,
    l_t = 0.5, l_x = 0.2, sigma = 1."""
    return heat_problem(16, 16, amps=np.array([1.0]), name="config0_heat1d_16x16")


def config1(seed: int = 1) -> Problem:
    """BASELINE.json configs[1]: 256 time x 512 space cells, IC = seeded sum
    of 8 sines with A_k ~ N(0, 1/k^2)."""
    return heat_problem(256, 512, amps=sine_series_ic(8, seed), name="config1_heat1d_256x512")


def heat_grid(nt: int, nx: int) -> Grid:
    """Dense prediction grid on [0,1]^2 (64x64 for config 0, 512x1024 for config 1)."""
    return Grid([np.linspace(0.0, 1.0, nt), np.linspace(0.0, 1.0, nx)], 0)


def _gauss_cell_integrals(lo, hi, c, w):
    """int_lo^hi exp(-(x-c)^2 / (2 w^2)) dx (closed form with erf)."""
    from scipy.special import erf
    s = np.sqrt(2.0) * w
    return w * np.sqrt(np.pi / 2.0) * (erf((hi - c) / s) - erf((lo - c) / s))


def _face_blocks(T, X, Y, ht, hx, hy, terms_for_face, jitter, deflate=True):
    """Four spatial boundary faces of a [0,1]^2 domain as FVM-style cell blocks:
    x=0 / x=1: (t cells) x point x (y cells);  y=0 / y=1: (t cells) x (x cells) x point y."""
    out = []
    for name, sites, h in [("BCx0", [T, point(0.0), Y], hy), ("BCx1", [T, point(1.0), Y], hy),
                           ("BCy0", [T, X, point(0.0)], hx), ("BCy1", [T, X, point(1.0)], hx)]:
        n = sites[0].n * sites[1].n * sites[2].n
        out.append(Block(name, sites, terms_for_face(name), jitter * (ht * h) ** 2, deflate, np.zeros(n)))
    return out


def wave_analytic_sine(c: float, t, x, y) -> np.ndarray:
    """u(t,x,y) = cos(sqrt(2) pi c t) sin(pi x) sin(pi y): the solution of
    u_tt = c^2 (u_xx + u_yy) on [0,1]^2 with u(0) = sin(pi x) sin(pi y),
    u_t(0) = 0, Dirichlet-0 (the i = j = 1 mode of PAPER.md l.703)."""
    t, x, y = np.broadcast_arrays(*np.ix_(np.asarray(t, float), np.asarray(x, float), np.asarray(y, float)))
    return np.cos(np.sqrt(2.0) * np.pi * c * t) * np.sin(np.pi * x) * np.sin(np.pi * y)


def wave_problem(nt: int, nx: int, ny: int, *, c: float = 1.0, ell=(0.1, 0.05, 0.05), q: int = 3,
                 centers=None, width: float = 0.05, seed: int = 2, jitter: float = 1e-8,
                 ic: str = "bump", name: str | None = None) -> Problem:
    """BASELINE config 2: u_tt = c^2 (u_xx + u_yy) on [0,1] x [0,1]^2, Matérn-7/2.
    IC cells: u(0,.) = Gaussian bump (seeded centre, width 0.05) and u_t(0,.) = 0;
    Dirichlet-0 BC cells on the four faces.  `centers` (k x 2) gives a k-RHS
    batch (the bump centres); the problem's rhs() is the first one, all k are
    in meta['rhs_batch']."""
    rng = np.random.default_rng(seed)
    if centers is None:
        centers = rng.uniform(0.3, 0.7, size=(4, 2))
    T, X, Y = cells(nt), cells(nx), cells(ny)
    ht, hx, hy = 1.0 / nt, 1.0 / nx, 1.0 / ny
    if ic == "sine":  # u(0,x,y) = sin(pi x) sin(pi y): exact cell integrals
        sx = (np.cos(np.pi * X.lo) - np.cos(np.pi * X.hi)) / np.pi
        sy = (np.cos(np.pi * Y.lo) - np.cos(np.pi * Y.hi)) / np.pi
        ic_vals = [np.outer(sx, sy).ravel()]
    else:
        ic_vals = [np.outer(_gauss_cell_integrals(X.lo, X.hi, cx, width),
                            _gauss_cell_integrals(Y.lo, Y.hi, cy, width)).ravel() for cx, cy in centers]
    blocks = [
        Block("IC_u", [point(0.0), X, Y], [Term(1.0, (0, 0, 0))], jitter * (hx * hy) ** 2, True, ic_vals[0]),
        Block("IC_ut", [point(0.0), X, Y], [Term(1.0, (1, 0, 0))], jitter * (hx * hy) ** 2, True,
              np.zeros(nx * ny)),
    ]
    blocks += _face_blocks(T, X, Y, ht, hx, hy, lambda f: [Term(1.0, (0, 0, 0))], jitter)
    blocks.append(Block("PDE", [T, X, Y], [Term(1.0, (2, 0, 0)), Term(-c * c, (0, 2, 0)), Term(-c * c, (0, 0, 2))],
                        0.0, False, np.zeros(nt * nx * ny)))
    kern = [[Kernel1D(q, ell[0]), Kernel1D(q, ell[1]), Kernel1D(q, ell[2])]]
    p = Problem(name or f"wave2d_{nt}x{nx}x{ny}", 3, kern, blocks, meta=dict(kind="wave2d", c=c, centers=centers))
    rhs_batch = []
    for v in ic_vals:
        rhs_batch.append(np.concatenate([v] + [b.rhs for b in blocks[1:]]))
    p.meta["rhs_batch"] = np.stack(rhs_batch)
    return p


def config2() -> Problem:
    """BASELINE.json configs[2]: 64 x 128 x 128 cells (~1.05M FVM obs), 4-RHS batch."""
    return wave_problem(64, 128, 128, name="config2_wave2d_64x128x128")


def advdiff_problem(nt: int, nx: int, ny: int, *, a=(1.0, 0.5), eps: float = 0.01, ell=(0.2, 0.1, 0.1),
                    q: int = 2, n_modes: int = 32, seed: int = 3, jitter: float = 1e-8,
                    name: str | None = None) -> Problem:
    """BASELINE config 3: u_t + a.grad u = eps Lap u on [0,1] x [0,1]^2, Matérn-5/2,
    seeded random-Fourier IC (n_modes sine modes, amplitudes ~ N(0, 1/|k|^2)),
    Dirichlet-0 BC cells."""
    rng = np.random.default_rng(seed)
    T, X, Y = cells(nt), cells(nx), cells(ny)
    ht, hx, hy = 1.0 / nt, 1.0 / nx, 1.0 / ny
    ks = rng.integers(1, 9, size=(n_modes, 2))
    amp = rng.standard_normal(n_modes) / np.sqrt((ks ** 2).sum(1))
    ix = lambda k, S: (np.cos(k * np.pi * S.lo) - np.cos(k * np.pi * S.hi)) / (k * np.pi)
    ic = sum(A * np.outer(ix(k1, X), ix(k2, Y)) for A, (k1, k2) in zip(amp, ks)).ravel()
    blocks = [Block("IC", [point(0.0), X, Y], [Term(1.0, (0, 0, 0))], jitter * (hx * hy) ** 2, True, ic)]
    blocks += _face_blocks(T, X, Y, ht, hx, hy, lambda f: [Term(1.0, (0, 0, 0))], jitter)
    blocks.append(Block("PDE", [T, X, Y], [Term(1.0, (1, 0, 0)), Term(a[0], (0, 1, 0)), Term(a[1], (0, 0, 1)),
                                         Term(-eps, (0, 2, 0)), Term(-eps, (0, 0, 2))],
                        0.0, False, np.zeros(nt * nx * ny)))
    kern = [[Kernel1D(q, ell[0]), Kernel1D(q, ell[1]), Kernel1D(q, ell[2])]]
    return Problem(name or f"advdiff2d_{nt}x{nx}x{ny}", 3, kern, blocks, meta=dict(kind="advdiff2d", a=a, eps=eps))


def config3() -> Problem:
    """BASELINE.json configs[3]: 128 x 256 x 256 cells (~8.4M FVM obs)."""
    return advdiff_problem(128, 256, 256, name="config3_advdiff2d_128x256x256")


def shallow_water_problem(nt: int, nx: int, ny: int, *, g: float = 9.81, H: float = 1.0,
                          ell=(0.2, 0.1, 0.1), q: int = 2, width: float = 0.08, noise_frac: float = 0.01,
                          seed: int = 4, jitter: float = 1e-8, center=None, name: str | None = None) -> Problem:
    """BASELINE config 4: linearised constant-depth shallow water (PAPER.md
    Eqs. 24-26 with f = k = 0, constant H):
        eta_t + H (u_x + v_y) = 0,   u_t + g eta_x = 0,   v_t + g eta_y = 0
    three outputs (eta, u, v) with independent Matérn-5/2 product priors
    (Eq. 17); per output the same cell grid.  IC cells: eta = seeded Gaussian
    displacement with 1% i.i.d. Gaussian observation noise (noise variance =
    (0.01 std(eta_IC))^2, values perturbed with the same draw), u = v = 0.
    Radiation BC cells on the four faces (App. C.4, P:l.757-761):
    eta_t -/+ c eta_n = 0 with c = sqrt(g H), sign per outward normal."""
    rng = np.random.default_rng(seed)
    T, X, Y = cells(nt), cells(nx), cells(ny)
    ht, hx, hy = 1.0 / nt, 1.0 / nx, 1.0 / ny
    cx, cy = rng.uniform(0.35, 0.65, size=2)
    if center is not None:  # fixed centre (e.g. (0.5, 0.5) for the mirror-symmetry pin)
        cx, cy = center
    eta0 = np.outer(_gauss_cell_integrals(X.lo, X.hi, cx, width), _gauss_cell_integrals(Y.lo, Y.hi, cy, width)).ravel()
    sd = noise_frac * float(np.std(eta0))
    eta_obs = eta0 + sd * rng.standard_normal(eta0.shape)
    ETA, U, V = 0, 1, 2
    blocks = [
        Block("IC_eta", [point(0.0), X, Y], [Term(1.0, (0, 0, 0), ETA)], sd * sd, True, eta_obs),
        Block("IC_u", [point(0.0), X, Y], [Term(1.0, (0, 0, 0), U)], jitter * (hx * hy) ** 2, True, np.zeros(nx * ny)),
        Block("IC_v", [point(0.0), X, Y], [Term(1.0, (0, 0, 0), V)], jitter * (hx * hy) ** 2, True, np.zeros(nx * ny)),
    ]
    c = float(np.sqrt(g * H))

    def rad(face):
        if face == "BCx0":
            return [Term(1.0, (1, 0, 0), ETA), Term(-c, (0, 1, 0), ETA)]
        if face == "BCx1":
            return [Term(1.0, (1, 0, 0), ETA), Term(c, (0, 1, 0), ETA)]
        if face == "BCy0":
            return [Term(1.0, (1, 0, 0), ETA), Term(-c, (0, 0, 1), ETA)]
        return [Term(1.0, (1, 0, 0), ETA), Term(c, (0, 0, 1), ETA)]

    blocks += _face_blocks(T, X, Y, ht, hx, hy, rad, jitter)
    n = nt * nx * ny
    blocks += [
        Block("PDE_eta", [T, X, Y], [Term(1.0, (1, 0, 0), ETA), Term(H, (0, 1, 0), U), Term(H, (0, 0, 1), V)],
              0.0, False, np.zeros(n)),
        Block("PDE_u", [T, X, Y], [Term(1.0, (1, 0, 0), U), Term(g, (0, 1, 0), ETA)], 0.0, False, np.zeros(n)),
        Block("PDE_v", [T, X, Y], [Term(1.0, (1, 0, 0), V), Term(g, (0, 0, 1), ETA)], 0.0, False, np.zeros(n)),
    ]
    kern = [[Kernel1D(q, ell[0]), Kernel1D(q, ell[1]), Kernel1D(q, ell[2])] for _ in range(3)]
    return Problem(name or f"shallow_water_{nt}x{nx}x{ny}", 3, kern, blocks,
                   meta=dict(kind="shallow_water", g=g, H=H, c=c))


def config4() -> Problem:
    """BASELINE.json configs[4]: 96 x 192 x 192 cells per output (~10.6M obs)."""
    return shallow_water_problem(96, 192, 192, name="config4_shallow_water_96x192x192")


def cos_ode_problem(n: int, q: int = 2, ell: float = 1.0) -> Problem:
    """PAPER.md Fig. 2 (l.166): du/dx = cos(x) on [0, 2 pi], u(0) = u(2 pi) = 0,
    n FVM cells; the cell observation int_a^b u' = u(b) - u(a) (Eq. 10) with
    right-hand side int_a^b cos = sin(b) - sin(a)."""
    X = cells(n, 0.0, 2 * np.pi)
    rhs = np.sin(X.hi) - np.sin(X.lo)
    blocks = [
        Block("BC", [points([0.0, 2 * np.pi])], [Term(1.0, (0,))], 1e-10, True, np.zeros(2)),
        Block("PDE", [X], [Term(1.0, (1,))], 0.0, False, rhs),
    ]
    return Problem(f"cos_ode_{n}", 1, [[Kernel1D(q, ell, 1.0)]], blocks, meta=dict(kind="cos_ode"))


def random_vectors(n: int, nrhs: int, seed: int) -> np.ndarray:
    """Seeded standard-normal block of vectors, shape (nrhs, n)."""
    return np.random.default_rng(seed).standard_normal((nrhs, n))
