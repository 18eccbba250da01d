"""Synthetic unit-cube meshes for the benchmark configurations.

Vectorized restatement of ``pkg/src/feklab/mesh.py:29-120`` that produces the
reference's element order and coordinates BIT FOR BIT (pinned against
``tests/golden/meshes.npz``) at numpy speed instead of a Python loop:

* tets (``mesh.py:49-68``): cell (ix, iy, iz) in C order, then the six Kuhn
  path tets in ``itertools.permutations(range(3))`` order; odd permutations
  swap vertices 1 and 2.  Every coordinate is either the cell origin
  ``i*h`` or ``i*h + h`` (the reference adds exact zeros for the other axes);
* prisms (``mesh.py:71-88``): base square (ix, iy) split into two triangles
  extruded from z=0 to z=1;
* coefficients: ``default_rng(seed).uniform(-1, 1, (n, DS))`` (``mesh.py:103-106``).

``jitter_top_faces`` makes prisms non-affine for configs C3-C5:
seeded in-plane ``U(-0.15, 0.15) * h`` offsets of the three top-face vertices.
"""

from __future__ import annotations

from dataclasses import dataclass
from itertools import permutations

import numpy as np

from .layout import ELEMENT_MAJOR, BatchLayout, ElementBatch
from .problems import ProblemClass
from .refelem import ElementType

_PERMS = list(permutations(range(3)))
_ODD = [int(round(np.linalg.det(np.eye(3)[list(p)]))) < 0 for p in _PERMS]


@dataclass(frozen=True)
class MeshSpec:
    nx: int
    ny: int
    nz: int
    element_type: ElementType

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise ValueError("subdivision counts must be >= 1")

    @property
    def n_elements(self) -> int:
        if self.element_type is ElementType.TETRAHEDRON:
            return 6 * self.nx * self.ny * self.nz
        return 2 * self.nx * self.ny


def spec_for_element_count(element_type: ElementType, n_elements: int) -> MeshSpec:
    """Smallest roughly-cubic spec with >= n_elements (``mesh.py:112-120``)."""
    if n_elements < 1:
        raise ValueError("element count must be >= 1")
    if element_type is ElementType.TETRAHEDRON:
        side = int(np.ceil((n_elements / 6.0) ** (1.0 / 3.0)))
        return MeshSpec(side, side, side, element_type)
    side = int(np.ceil(np.sqrt(n_elements / 2.0)))
    return MeshSpec(side, side, 1, element_type)


def _tet_rows(spec: MeshSpec, cells: slice | None = None) -> np.ndarray:
    h = np.array([1.0 / spec.nx, 1.0 / spec.ny, 1.0 / spec.nz])
    ncell = spec.nx * spec.ny * spec.nz
    cell = np.arange(ncell)[cells] if cells is not None else np.arange(ncell)
    ix, rem = np.divmod(cell, spec.ny * spec.nz)
    iy, iz = np.divmod(rem, spec.nz)
    origin = np.stack([ix * h[0], iy * h[1], iz * h[2]], axis=1)  # (c, 3): int*float like the reference
    upper = origin + h                                           # origin + h, component-wise
    rows = np.empty((cell.size, 6, 4, 3))
    for p, (perm, odd) in enumerate(zip(_PERMS, _ODD)):
        stepped = np.zeros(3, dtype=bool)
        verts = [origin]
        for axis in perm:
            stepped = stepped.copy()
            stepped[axis] = True
            verts.append(np.where(stepped, upper, origin))
        if odd:
            verts[1], verts[2] = verts[2], verts[1]
        rows[:, p] = np.stack(verts, axis=1)
    return rows.reshape(-1, 12)


def _prism_rows(spec: MeshSpec, cells: slice | None = None) -> np.ndarray:
    hx, hy = 1.0 / spec.nx, 1.0 / spec.ny
    cell = np.arange(spec.nx * spec.ny)
    ix, iy = np.divmod(cell[cells] if cells is not None else cell, spec.ny)
    x0, y0 = ix * hx, iy * hy
    x1, y1 = x0 + hx, y0 + hy
    tris = (((x0, y0), (x1, y0), (x0, y1)), ((x1, y0), (x1, y1), (x0, y1)))
    rows = np.empty((x0.size, 2, 6, 3))
    for t, tri in enumerate(tris):
        for v, (x, y) in enumerate(tri):
            rows[:, t, v, 0] = x
            rows[:, t, v, 1] = y
            rows[:, t, v, 2] = 0.0
            rows[:, t, v + 3, 0] = x
            rows[:, t, v + 3, 1] = y
            rows[:, t, v + 3, 2] = 1.0
    return rows.reshape(-1, 18)


def node_count(spec: MeshSpec) -> int:
    """Vertices of the structured unit-cube mesh: (nx+1)(ny+1)(nz+1) grid points (tets) or the
    (nx+1)(ny+1) base points at z = 0 and z = 1 (prisms)."""
    if spec.element_type is ElementType.TETRAHEDRON:
        return (spec.nx + 1) * (spec.ny + 1) * (spec.nz + 1)
    return (spec.nx + 1) * (spec.ny + 1) * 2


def element_nodes(spec: MeshSpec) -> np.ndarray:
    """(n, nv) int32 global node numbers of every element, in geometry_rows' element and vertex
    order: the connectivity a matrix-free apply scatters through (kernels/apply.py).  The
    reference's batches carry coordinates only; for its structured meshes the topology is the
    grid's -- tets: the Kuhn path from the cell origin, prisms: the two base triangles extruded.
    (Top-face jitter moves coordinates, not connectivity.)"""
    if spec.element_type is ElementType.TETRAHEDRON:
        nx, ny, nz = spec.nx, spec.ny, spec.nz
        cell = np.arange(nx * ny * nz, dtype=np.int64)
        ix, rem = np.divmod(cell, ny * nz)
        iy, iz = np.divmod(rem, nz)
        out = np.empty((cell.size, 6, 4), dtype=np.int64)
        node = lambda dx, dy, dz: ((ix + dx) * (ny + 1) + (iy + dy)) * (nz + 1) + (iz + dz)  # noqa: E731
        for p, (perm, odd) in enumerate(zip(_PERMS, _ODD)):
            step = [0, 0, 0]
            verts = [node(0, 0, 0)]
            for axis in perm:
                step[axis] = 1
                verts.append(node(*step))
            if odd:
                verts[1], verts[2] = verts[2], verts[1]
            out[:, p] = np.stack(verts, axis=1)
        return out.reshape(-1, 4).astype(np.int32)
    nx, ny = spec.nx, spec.ny
    cell = np.arange(nx * ny, dtype=np.int64)
    ix, iy = np.divmod(cell, ny)
    base = lambda dx, dy: ((ix + dx) * (ny + 1) + (iy + dy)) * 2  # noqa: E731
    tris = (((0, 0), (1, 0), (0, 1)), ((1, 0), (1, 1), (0, 1)))
    out = np.empty((cell.size, 2, 6), dtype=np.int64)
    for t, tri in enumerate(tris):
        for v, (dx, dy) in enumerate(tri):
            out[:, t, v] = base(dx, dy)
            out[:, t, v + 3] = base(dx, dy) + 1
    return out.reshape(-1, 6).astype(np.int32)


def geometry_rows(spec: MeshSpec) -> np.ndarray:
    if spec.element_type is ElementType.TETRAHEDRON:
        return _tet_rows(spec)
    return _prism_rows(spec)


def coefficient_rows(n: int, problem: ProblemClass, element_type: ElementType, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(n, problem.coefficient_size(element_type)))


def jitter_top_faces(rows: np.ndarray, spec: MeshSpec, seed: int, amplitude: float = 0.15) -> np.ndarray:
    """Non-affine prisms: move top vertices 3..5 in-plane by U(-a, a) * (hx, hy).

    Draw order: ``default_rng(seed).uniform(-1, 1, (n, 3, 2))``.  With
    ``a = 0.15`` det J stays positive at every quadrature point.
    """
    if spec.element_type is not ElementType.PRISM:
        raise ValueError("top-face jitter applies to prisms")
    h = np.array([1.0 / spec.nx, 1.0 / spec.ny])
    rng = np.random.default_rng(seed)
    off = rng.uniform(-1.0, 1.0, size=(rows.shape[0], 3, 2)) * (amplitude * h)
    out = rows.reshape(-1, 6, 3).copy()
    out[:, 3:, :2] += off
    return out.reshape(-1, 18)


def generate_mesh(spec: MeshSpec, coeff_seed: int, problem: ProblemClass, layout: BatchLayout = ELEMENT_MAJOR,
                  pad_value: float = np.nan, jitter_seed: int | None = None) -> ElementBatch:
    """``feklab.mesh.generate_mesh`` plus optional prism top-face jitter."""
    geo = geometry_rows(spec)
    if jitter_seed is not None:
        geo = jitter_top_faces(geo, spec, jitter_seed)
    cof = coefficient_rows(spec.n_elements, problem, spec.element_type, coeff_seed)
    return ElementBatch.from_arrays(spec.element_type, problem, geo, cof, layout, pad_value)


# ---------------------------------------------------------------------------
# benchmark configurations (BASELINE.json "configs")
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class BenchConfig:
    key: str
    spec: MeshSpec
    problem: ProblemClass
    coeff_seed: int
    jitter_seed: int | None
    text: str


def bench_configs() -> dict[str, BenchConfig]:
    T, P = ElementType.TETRAHEDRON, ElementType.PRISM
    return {
        "C1": BenchConfig("C1", spec_for_element_count(T, 1_000_000), ProblemClass.POISSON, 0, None,
                          "Poisson on 1M linear tetrahedra, fp64"),
        "C2": BenchConfig("C2", spec_for_element_count(T, 4_000_000), ProblemClass.CONV_DIFF, 0, None,
                          "Generalized convection-diffusion-reaction on 4M linear tetrahedra, fp64"),
        "C3": BenchConfig("C3", MeshSpec(1415, 1415, 1, P), ProblemClass.POISSON, 0, 1,
                          "Poisson on 4M non-affine linear prisms, fp64"),
        "C4": BenchConfig("C4", MeshSpec(2829, 2829, 1, P), ProblemClass.CONV_DIFF, 0, 1,
                          "Convection-diffusion-reaction on 16M non-affine linear prisms"),
        "C5T": BenchConfig("C5T", MeshSpec(175, 175, 175, T), ProblemClass.CONV_DIFF, 0, None,
                           "C5 tet part: 32.2M tets, convection-diffusion-reaction"),
        "C5P": BenchConfig("C5P", MeshSpec(4000, 4000, 1, P), ProblemClass.CONV_DIFF, 1, 2,
                           "C5 prism part: 32M non-affine prisms, convection-diffusion-reaction"),
    }


def config_rows(cfg: BenchConfig) -> tuple[np.ndarray, np.ndarray]:
    geo = geometry_rows(cfg.spec)
    if cfg.jitter_seed is not None:
        geo = jitter_top_faces(geo, cfg.spec, cfg.jitter_seed)
    return geo, coefficient_rows(cfg.spec.n_elements, cfg.problem, cfg.spec.element_type, cfg.coeff_seed)


def config_window(cfg: BenchConfig, n: int) -> tuple[np.ndarray, np.ndarray]:
    """Host rows of the FIRST n elements of a configuration, without generating the rest.

    Element order is cell-major (6 tets / 2 prisms per cell) and every random stream is
    drawn row by row, so these are exactly rows [0, n) of ``config_rows(cfg)``.
    """
    spec = cfg.spec
    n = min(int(n), spec.n_elements)
    per_cell = 6 if spec.element_type is ElementType.TETRAHEDRON else 2
    cells = slice(0, -(-n // per_cell))
    rows_fn = _tet_rows if spec.element_type is ElementType.TETRAHEDRON else _prism_rows
    geo = rows_fn(spec, cells)[:n]
    if cfg.jitter_seed is not None:
        h = np.array([1.0 / spec.nx, 1.0 / spec.ny])
        off = np.random.default_rng(cfg.jitter_seed).uniform(-1.0, 1.0, size=(n, 3, 2)) * (0.15 * h)
        geo = geo.reshape(-1, 6, 3).copy()
        geo[:, 3:, :2] += off
        geo = geo.reshape(-1, 18)
    return geo, coefficient_rows(n, cfg.problem, spec.element_type, cfg.coeff_seed)


# ---------------------------------------------------------------------------
# device-side generation (libfek fek_mesh_geometry / fek_pcg64_uniform)
# ---------------------------------------------------------------------------

def pcg64_words(seed: int):
    """numpy PCG64(seed) state as the 4-word array fek_pcg64_uniform takes."""
    import ctypes

    st = np.random.PCG64(seed).state["state"]
    mask = (1 << 64) - 1
    words = [(st["state"] >> 64) & mask, st["state"] & mask, (st["inc"] >> 64) & mask, st["inc"] & mask]
    return (ctypes.c_ulonglong * 4)(*words)


def device_geometry(spec: MeshSpec, first: int = 0, n: int | None = None, jitter_seed: int | None = None,
                    amplitude: float = 0.15, device=None):
    """Geometry rows of elements [first, first+n) generated in HBM (flat float64 tensor).

    Bit-identical to ``geometry_rows(spec)[first:first+n]`` (plus
    ``jitter_top_faces(..., jitter_seed)``); no host work.
    """
    import torch

    from . import _native

    n = spec.n_elements - first if n is None else n
    out = torch.empty(n * spec.element_type.geometry_size, dtype=torch.float64, device=device or "cuda")
    lib = _native.load()
    js = pcg64_words(jitter_seed) if jitter_seed is not None else None
    code = _native.ELEMENT[spec.element_type.value]
    with torch.cuda.device(out.device):
        _native.check(lib.fek_mesh_geometry(code, spec.nx, spec.ny, spec.nz, first, n, js, amplitude,
                                            out.data_ptr(), torch.cuda.current_stream().cuda_stream),
                      "fek_mesh_geometry")
    return out


def device_coefficients(problem: ProblemClass, element_type: ElementType, seed: int, first: int, n: int,
                        device=None):
    """Coefficient rows [first, first+n) of ``coefficient_rows(..., seed)`` generated in HBM."""
    import torch

    from . import _native

    ds = problem.coefficient_size(element_type)
    out = torch.empty(n * ds, dtype=torch.float64, device=device or "cuda")
    lib = _native.load()
    with torch.cuda.device(out.device):
        _native.check(lib.fek_pcg64_uniform(pcg64_words(seed), first * ds, n * ds, -1.0, 1.0, out.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream), "fek_pcg64_uniform")
    return out


def device_config(cfg: BenchConfig, first: int = 0, n: int | None = None, device=None):
    """(geometry, coefficients) flat float64 CUDA tensors of elements [first, first+n) of a config."""
    n = cfg.spec.n_elements - first if n is None else n
    geo = device_geometry(cfg.spec, first, n, cfg.jitter_seed, device=device)
    cof = device_coefficients(cfg.problem, cfg.spec.element_type, cfg.coeff_seed, first, n, device=device)
    return geo, cof
