"""Host data model mirroring the reference form/action API (femsched, form.hpp).

Same names, argument meaning and validation messages as the reference so that
tests read like the reference's own tests:

  ScalarSpace / VectorSpace / FormSignature   form.hpp:71-148
  simplex_space_dim / usable_flops            form.hpp:151-173
  PointwiseMap (builder + DAG)                form.hpp:192-318
  Tabulations / IndexMap / MeshConnectivity   form.hpp:37-65, 324-405
  ProblemInstance                             form.hpp:407-435
  preset_signature / preset_map               form.hpp:625-734
  SynthRng / chain_index_map / make_problem   form.hpp:741-852
  generic_map / synthesize_problem            form.hpp:857-881

Arrays are numpy (float64 / int32).  Synthesis is vectorised: splitmix64 is a
counter-based generator (draw k is mix(seed0 + k*golden)), so make_problem
reproduces the reference's sequential draw order bit-for-bit without a Python
loop (pinned against the compiled reference in tests/test_oracle.py).

The B200 compute path is NOT here: `ProblemInstance.to_c()` produces the flat
descriptor that crosses the C-ABI (include/femgpu.h) into libfemgpu.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import abi

SUBGROUP_SIZE = 32  # kSubgroupSize, form.hpp:19


class InfeasibleError(RuntimeError):
    """femsched::InfeasibleError (form.hpp:24-26)."""


class VerificationError(RuntimeError):
    """femsched::VerificationError (form.hpp:29-31)."""


def ceil_div(a: int, b: int) -> int:
    return (a + b - 1) // b


# --------------------------------------------------------------------------- signature


@dataclass
class ScalarSpace:
    dofs: int = 0
    deriv_terms: int = 0


@dataclass
class VectorSpace:
    dofs: int = 0
    deriv_terms: int = 0
    components: List[int] = field(default_factory=list)


@dataclass
class FormSignature:
    dim: int = 2
    scalar_spaces: List[ScalarSpace] = field(default_factory=list)
    vector_spaces: List[VectorSpace] = field(default_factory=list)
    test_dofs: int = 0
    test_deriv_terms: int = 0
    quad_points: int = 0
    coord_dofs: int = 0
    affine_geometry: bool = True
    coordinate_space: int = -1
    word_bytes: int = 8

    def trial_space_count(self) -> int:
        return len(self.scalar_spaces) + len(self.vector_spaces)

    def scalar_term_offset(self, space: int) -> int:
        return sum(s.deriv_terms for s in self.scalar_spaces[:space])

    def vector_term_offset(self, space: int) -> int:
        return sum(v.deriv_terms for v in self.vector_spaces[:space])

    def total_scalar_terms(self) -> int:
        return self.scalar_term_offset(len(self.scalar_spaces))

    def total_vector_terms(self) -> int:
        return self.vector_term_offset(len(self.vector_spaces))

    def validate(self) -> None:  # form.hpp:115-147
        if self.dim < 1 or self.dim > 3:
            raise ValueError("signature: dim must be 1..3")
        if not self.scalar_spaces and not self.vector_spaces:
            raise ValueError("signature: at least one trial space required")
        if self.quad_points < 1:
            raise ValueError("signature: quad_points must be >= 1")
        if self.test_dofs < 1 or self.test_deriv_terms < 1:
            raise ValueError("signature: test space counts must be positive")
        if self.word_bytes not in (4, 8):
            raise ValueError("signature: word_bytes must be 4 or 8")
        for s in self.scalar_spaces:
            if s.dofs < 1 or s.deriv_terms < 1:
                raise ValueError("signature: scalar space counts must be positive")
        for v in self.vector_spaces:
            if v.dofs < 1 or v.deriv_terms < 1:
                raise ValueError("signature: vector space counts must be positive")
            if len(v.components) != v.deriv_terms:
                raise ValueError("signature: one component index per derivative term required")
            for c in v.components:
                if c < 0 or c >= self.dim:
                    raise ValueError("signature: component index out of range")
        if self.affine_geometry:
            if self.coord_dofs != self.dim + 1:
                raise ValueError("signature: affine geometry requires coord_dofs == dim+1")
            if self.coordinate_space != -1:
                raise ValueError("signature: coordinate_space is only meaningful when non-affine")
        elif self.coordinate_space < 0 or self.coordinate_space >= len(self.vector_spaces):
            raise ValueError("signature: non-affine geometry requires the coordinate space to appear in "
                             "the vector-space list exactly once")


def simplex_space_dim(degree: int, d: int) -> int:  # form.hpp:151-160
    if degree < 0 or d < 1 or d > 3:
        raise ValueError("simplex_space_dim: degree >= 0 and d in 1..3 required")
    num = den = 1
    for i in range(1, d + 1):
        num *= degree + i
        den *= i
    return num // den


def usable_flops(sig: FormSignature) -> int:  # form.hpp:164-173
    sig.validate()
    ops = 0
    for s in sig.scalar_spaces:
        ops += 2 * s.deriv_terms * sig.quad_points * s.dofs
    for v in sig.vector_spaces:
        ops += 2 * v.deriv_terms * sig.quad_points * v.dofs
    ops += 2 * sig.test_deriv_terms * sig.quad_points * sig.test_dofs
    return ops


# --------------------------------------------------------------------------- pointwise map


class PointwiseMap:
    """Add/multiply/constant DAG, one output per test derivative term (form.hpp:192-318)."""

    CONSTANT, SCALAR_DERIV, VECTOR_DERIV, JACOBIAN, DETERMINANT, WEIGHT, COORD, ADD, MUL, INV_JACOBIAN = range(10)

    def __init__(self):
        self.nodes: list = []  # (op, value, a, b)
        self.outputs: list = []

    def _push(self, op, value=0.0, a=-1, b=-1) -> int:
        self.nodes.append((op, float(value), a, b))
        return len(self.nodes) - 1

    def constant(self, v): return self._push(self.CONSTANT, v)
    def scalar_deriv(self, space, term): return self._push(self.SCALAR_DERIV, 0.0, space, term)
    def vector_deriv(self, space, term): return self._push(self.VECTOR_DERIV, 0.0, space, term)
    def jacobian(self, row, col): return self._push(self.JACOBIAN, 0.0, row, col)
    def inverse_jacobian(self, row, col): return self._push(self.INV_JACOBIAN, 0.0, row, col)  # extension
    def determinant(self): return self._push(self.DETERMINANT)
    def weight(self): return self._push(self.WEIGHT)
    def coord(self, vertex, axis): return self._push(self.COORD, 0.0, vertex, axis)
    def add(self, x, y): return self._push(self.ADD, 0.0, x, y)
    def mul(self, x, y): return self._push(self.MUL, 0.0, x, y)

    def sub(self, x, y):
        """x - y as x + (-1)*y (the map language has no subtraction)."""
        return self.add(x, self.mul(self.constant(-1.0), y))

    def sum(self, terms: Sequence[int]) -> int:
        if not terms:
            return self.constant(0.0)
        acc = terms[0]
        for t in terms[1:]:
            acc = self.add(acc, t)
        return acc

    def add_output(self, node: int) -> None:
        self.outputs.append(node)

    def output_count(self) -> int:
        return len(self.outputs)

    def validate(self, sig: FormSignature) -> None:  # form.hpp:234-280
        if len(self.outputs) != sig.test_deriv_terms:
            raise ValueError("pointwise map: one expression per test derivative term required")
        for out in self.outputs:
            if out < 0 or out >= len(self.nodes):
                raise ValueError("pointwise map: output references unknown node")
        for idx, (op, _v, a, b) in enumerate(self.nodes):
            if op == self.SCALAR_DERIV:
                if a < 0 or a >= len(sig.scalar_spaces) or b < 0 or b >= sig.scalar_spaces[a].deriv_terms:
                    raise ValueError("pointwise map: undeclared scalar derivative input")
            elif op == self.VECTOR_DERIV:
                if a < 0 or a >= len(sig.vector_spaces) or b < 0 or b >= sig.vector_spaces[a].deriv_terms:
                    raise ValueError("pointwise map: undeclared vector derivative input")
            elif op in (self.JACOBIAN, self.INV_JACOBIAN):
                if not sig.affine_geometry:
                    raise ValueError("pointwise map: jacobian input requires affine geometry")
                if a < 0 or a >= sig.dim or b < 0 or b >= sig.dim:
                    raise ValueError("pointwise map: jacobian index out of range")
            elif op == self.DETERMINANT:
                if not sig.affine_geometry:
                    raise ValueError("pointwise map: determinant input requires affine geometry")
            elif op == self.COORD:
                if not sig.affine_geometry:
                    raise ValueError("pointwise map: coord input requires affine geometry")
                if a < 0 or a >= sig.coord_dofs or b < 0 or b >= sig.dim:
                    raise ValueError("pointwise map: coord index out of range")
            elif op in (self.ADD, self.MUL):
                if a < 0 or b < 0 or a >= idx or b >= idx:
                    raise ValueError("pointwise map: child must precede its parent")

    def copy(self) -> "PointwiseMap":
        m = PointwiseMap()
        m.nodes = list(self.nodes)
        m.outputs = list(self.outputs)
        return m


# --------------------------------------------------------------------------- data


@dataclass
class IndexMap:
    """int32 [cell][entry] map into a global array of global_count (form.hpp:49-65)."""
    indices: np.ndarray  # shape (cells, entries), int32
    global_count: int

    @property
    def cells(self) -> int:
        return int(self.indices.shape[0])

    @property
    def entries(self) -> int:
        return int(self.indices.shape[1])


@dataclass
class Tabulations:
    scalar_phi: List[np.ndarray] = field(default_factory=list)  # [space] (terms, Q, dofs)
    vector_phi: List[np.ndarray] = field(default_factory=list)  # [space] (terms, Q, dofs)
    psi: Optional[np.ndarray] = None                             # (terms, test_dofs, Q)
    weights: Optional[np.ndarray] = None                         # (Q,)


@dataclass
class MeshConnectivity:
    cell_count: int = 0
    scalar_maps: List[IndexMap] = field(default_factory=list)
    vector_maps: List[IndexMap] = field(default_factory=list)
    test_map: Optional[IndexMap] = None
    coord_map: Optional[IndexMap] = None
    coords: Optional[np.ndarray] = None  # (coord_global_count, dim)
    coord_global_count: int = 0


@dataclass
class ProblemInstance:
    signature: FormSignature
    map: PointwiseMap
    tabulations: Tabulations
    connectivity: MeshConnectivity
    scalar_inputs: List[np.ndarray] = field(default_factory=list)
    vector_inputs: List[np.ndarray] = field(default_factory=list)  # (global*dim,) interleaved
    output_size: int = 0

    def validate(self) -> None:
        """Structural part of ProblemInstance::validate (form.hpp:416-434); the
        O(size) bounds/finiteness checks run natively in femgpu_validate."""
        sig = self.signature
        sig.validate()
        self.map.validate(sig)
        tab, conn = self.tabulations, self.connectivity
        if len(tab.scalar_phi) != len(sig.scalar_spaces) or len(tab.vector_phi) != len(sig.vector_spaces):
            raise ValueError("tabulations: one phi set per trial space required")
        for s, phi in zip(sig.scalar_spaces, tab.scalar_phi):
            if phi.shape != (s.deriv_terms, sig.quad_points, s.dofs):
                raise ValueError("tabulations: scalar phi shape mismatch")
        for v, phi in zip(sig.vector_spaces, tab.vector_phi):
            if phi.shape != (v.deriv_terms, sig.quad_points, v.dofs):
                raise ValueError("tabulations: vector phi shape mismatch")
        if tab.psi is None or tab.psi.shape != (sig.test_deriv_terms, sig.test_dofs, sig.quad_points):
            raise ValueError("tabulations: psi shape mismatch")
        if tab.weights is None or tab.weights.shape != (sig.quad_points,):
            raise ValueError("tabulations: weight count mismatch")
        if conn.cell_count < 1:
            raise ValueError("connectivity: at least one cell required")
        if len(conn.scalar_maps) != len(sig.scalar_spaces) or len(conn.vector_maps) != len(sig.vector_spaces):
            raise ValueError("connectivity: one index map per trial space required")
        for m, s in zip(conn.scalar_maps, sig.scalar_spaces):
            if m.indices.shape != (conn.cell_count, s.dofs):
                raise ValueError("connectivity: bad shape for scalar space map")
        for m, v in zip(conn.vector_maps, sig.vector_spaces):
            if m.indices.shape != (conn.cell_count, v.dofs):
                raise ValueError("connectivity: bad shape for vector space map")
        if conn.test_map is None or conn.test_map.indices.shape != (conn.cell_count, sig.test_dofs):
            raise ValueError("connectivity: bad shape for test space map")
        if sig.affine_geometry:
            if conn.coord_map is None or conn.coord_map.indices.shape != (conn.cell_count, sig.coord_dofs):
                raise ValueError("connectivity: bad shape for coordinate map")
            if conn.coord_global_count < 1 or conn.coords is None or \
                    conn.coords.size != conn.coord_global_count * sig.dim:
                raise ValueError("connectivity: coordinate array shape mismatch")
            if conn.coord_map.global_count != conn.coord_global_count:
                raise ValueError("connectivity: coordinate map bound mismatch")
        if len(self.scalar_inputs) != len(sig.scalar_spaces) or len(self.vector_inputs) != len(sig.vector_spaces):
            raise ValueError("instance: one input vector per trial space required")
        for x, m in zip(self.scalar_inputs, conn.scalar_maps):
            if x.size != m.global_count:
                raise ValueError("instance: scalar input length mismatch")
        for x, m in zip(self.vector_inputs, conn.vector_maps):
            if x.size != m.global_count * sig.dim:
                raise ValueError("instance: vector input length mismatch")
        if self.output_size != conn.test_map.global_count:
            raise ValueError("instance: output length mismatch")

    # ---------------------------------------------------------------- C-ABI
    def to_c(self) -> "CProblem":
        return CProblem(self)

    def copy(self) -> "ProblemInstance":
        import copy
        return copy.deepcopy(self)


class CProblem:
    """Keeps the numpy buffers alive while a femgpu_problem points into them."""

    def __init__(self, p: ProblemInstance):
        sig, tab, conn = p.signature, p.tabulations, p.connectivity
        keep = []

        def f64(a):
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return a

        def i32(a):
            a = np.ascontiguousarray(a, dtype=np.int32)
            keep.append(a)
            return a

        ns, nv = len(sig.scalar_spaces), len(sig.vector_spaces)
        if ns > abi.MAX_SPACES or nv > abi.MAX_SPACES:
            raise ValueError("instance: at most %d scalar and %d vector spaces" % (abi.MAX_SPACES, abi.MAX_SPACES))
        sarr = (abi.Space * max(ns, 1))()
        varr = (abi.Space * max(nv, 1))()
        for i, s in enumerate(sig.scalar_spaces):
            sp = sarr[i]
            sp.dofs, sp.deriv_terms = s.dofs, s.deriv_terms
            sp.components = None
            sp.phi = abi.dptr(f64(tab.scalar_phi[i]))
            sp.map = abi.iptr(i32(conn.scalar_maps[i].indices))
            sp.global_count = conn.scalar_maps[i].global_count
            sp.input = abi.dptr(f64(p.scalar_inputs[i]))
        for i, v in enumerate(sig.vector_spaces):
            sp = varr[i]
            sp.dofs, sp.deriv_terms = v.dofs, v.deriv_terms
            sp.components = abi.iptr(i32(np.asarray(v.components, dtype=np.int32)))
            sp.phi = abi.dptr(f64(tab.vector_phi[i]))
            sp.map = abi.iptr(i32(conn.vector_maps[i].indices))
            sp.global_count = conn.vector_maps[i].global_count
            sp.input = abi.dptr(f64(p.vector_inputs[i]))
        nodes = (abi.MapNode * max(len(p.map.nodes), 1))()
        for i, (op, val, a, b) in enumerate(p.map.nodes):
            nodes[i].op, nodes[i].value, nodes[i].a, nodes[i].b = op, val, a, b
        outs = i32(np.asarray(p.map.outputs, dtype=np.int32).reshape(-1))
        d = abi.Problem()
        d.dim, d.quad_points, d.coord_dofs = sig.dim, sig.quad_points, sig.coord_dofs
        d.affine_geometry, d.coordinate_space, d.word_bytes = int(sig.affine_geometry), sig.coordinate_space, sig.word_bytes
        d.n_scalar, d.n_vector = ns, nv
        d.scalar_spaces, d.vector_spaces = sarr, varr
        d.test_dofs, d.test_deriv_terms = sig.test_dofs, sig.test_deriv_terms
        d.psi = abi.dptr(f64(tab.psi))
        d.weights = abi.dptr(f64(tab.weights))
        d.cell_count = conn.cell_count
        d.test_global_count = conn.test_map.global_count
        d.test_map = abi.iptr(i32(conn.test_map.indices))
        if sig.affine_geometry:
            d.coord_map = abi.iptr(i32(conn.coord_map.indices))
            d.coords = abi.dptr(f64(conn.coords))
            d.coord_global_count = conn.coord_global_count
        d.n_map_nodes = len(p.map.nodes)
        d.map_nodes = nodes
        d.map_outputs = abi.iptr(outs)
        d.n_map_outputs = len(p.map.outputs)
        d.output_size = p.output_size
        self.desc = d
        self._keep = (keep, sarr, varr, nodes)

    def ref(self):
        return C.byref(self.desc)


# --------------------------------------------------------------------------- presets

OPERATORS = ("mass", "laplace", "helmholtz", "elasticity", "hyperelasticity")


def operator_from_name(name: str) -> str:  # form.hpp:614-621
    if name == "poisson":
        return "laplace"
    if name in OPERATORS:
        return name
    raise ValueError("unknown operator preset: " + name)


def preset_signature(op: str, dim: int, degree: int, quad_points: int) -> FormSignature:  # form.hpp:625-671
    op = operator_from_name(op)
    vector_valued = op in ("elasticity", "hyperelasticity")
    if dim < 1 or dim > 3 or (vector_valued and dim < 2):
        raise ValueError("preset_signature: unsupported operator/dimension combination")
    if degree < 1:
        raise ValueError("preset_signature: degree >= 1 required")
    if quad_points < 1:
        raise ValueError("preset_signature: quad_points >= 1 required")
    n = simplex_space_dim(degree, dim)
    sig = FormSignature(dim=dim, quad_points=quad_points, coord_dofs=dim + 1, affine_geometry=True, word_bytes=8)
    if op == "mass":
        sig.scalar_spaces = [ScalarSpace(n, 1)]
        sig.test_dofs, sig.test_deriv_terms = n, 1
    elif op == "laplace":
        sig.scalar_spaces = [ScalarSpace(n, dim)]
        sig.test_dofs, sig.test_deriv_terms = n, dim
    elif op == "helmholtz":
        sig.scalar_spaces = [ScalarSpace(n, dim + 1)]
        sig.test_dofs, sig.test_deriv_terms = n, dim + 1
    else:
        comps = [a for a in range(dim) for _c in range(dim)]
        sig.vector_spaces = [VectorSpace(n, dim * dim, comps)]
        sig.test_dofs, sig.test_deriv_terms = n * dim, dim * dim
    sig.validate()
    return sig


def _metric_entry(m: PointwiseMap, d: int, r: int, c: int) -> int:  # (J^T J)[r][c], form.hpp:681-685
    return m.sum([m.mul(m.jacobian(k, r), m.jacobian(k, c)) for k in range(d)])


def preset_map(op: str, sig: FormSignature) -> PointwiseMap:  # form.hpp:676-734
    op = operator_from_name(op)
    m = PointwiseMap()
    d = sig.dim
    wd = m.mul(m.weight(), m.determinant())
    if op == "mass":
        m.add_output(m.mul(wd, m.scalar_deriv(0, 0)))
    elif op in ("laplace", "helmholtz"):
        for r in range(d):
            terms = [m.mul(_metric_entry(m, d, r, c), m.scalar_deriv(0, c)) for c in range(d)]
            m.add_output(m.mul(wd, m.sum(terms)))
        if op == "helmholtz":
            m.add_output(m.mul(wd, m.scalar_deriv(0, d)))
    elif op == "elasticity":
        for a in range(d):
            for c in range(d):
                sym = m.add(m.vector_deriv(0, a * d + c), m.vector_deriv(0, c * d + a))
                m.add_output(m.mul(wd, m.mul(m.constant(0.5), sym)))
    else:  # hyperelasticity (linear lambda/mu map)
        lam, mu = 1.25, 0.75
        trace = m.sum([m.vector_deriv(0, k * d + k) for k in range(d)])
        for a in range(d):
            for c in range(d):
                sym = m.add(m.vector_deriv(0, a * d + c), m.vector_deriv(0, c * d + a))
                term = m.mul(m.constant(mu), sym)
                if a == c:
                    term = m.add(term, m.mul(m.constant(lam), trace))
                m.add_output(m.mul(wd, term))
    m.validate(sig)
    return m


def generic_map(sig: FormSignature) -> PointwiseMap:  # form.hpp:857-876
    m = PointwiseMap()
    scale = m.weight()
    if sig.affine_geometry:
        scale = m.mul(scale, m.determinant())
    for k in range(sig.test_deriv_terms):
        terms = []
        v = 0
        for i, s in enumerate(sig.scalar_spaces):
            for t in range(s.deriv_terms):
                terms.append(m.mul(m.constant(1.0 + ((k * 7 + v * 3) % 5) * 0.25), m.scalar_deriv(i, t)))
                v += 1
        for i, vs in enumerate(sig.vector_spaces):
            for t in range(vs.deriv_terms):
                terms.append(m.mul(m.constant(1.0 + ((k * 7 + v * 3) % 5) * 0.25), m.vector_deriv(i, t)))
                v += 1
        m.add_output(m.mul(scale, m.sum(terms)))
    m.validate(sig)
    return m


# --------------------------------------------------------------------------- synthesis

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK64 = (1 << 64) - 1


class SynthRng:
    """splitmix64 (form.hpp:741-757), vectorised: draws() returns the next n outputs."""

    def __init__(self, seed: int):
        self.state = int(seed) & _MASK64

    def draws(self, n: int) -> np.ndarray:
        k = np.arange(1, n + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + k * _GOLDEN
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * 0x9E3779B97F4A7C15) & _MASK64
        return z

    def draws_at(self, idx: np.ndarray) -> np.ndarray:
        """The outputs at stream positions idx (0 = the next draw) without advancing: splitmix64 is
        counter-based, so one rank of a partitioned run draws only the entries of its own nodes."""
        k = np.asarray(idx, dtype=np.uint64) + np.uint64(1)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + k * _GOLDEN
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
        return z

    def skip(self, n: int) -> None:
        self.state = (self.state + n * 0x9E3779B97F4A7C15) & _MASK64

    def uniform_at(self, lo: float, span: float, idx: np.ndarray) -> np.ndarray:
        return uniform_from_raw(lo, span, (self.draws_at(idx) >> np.uint64(11)).astype(np.float64))

    def next_u64(self) -> int:
        return int(self.draws(1)[0])

    def raw53(self, n: int) -> np.ndarray:
        """next_u64() >> 11 as float64 (exact: < 2^53)."""
        return (self.draws(n) >> np.uint64(11)).astype(np.float64)

    def uniform(self, lo: float, span: float, n: int) -> np.ndarray:
        return uniform_from_raw(lo, span, self.raw53(n))


def uniform_from_raw(lo: float, span: float, raw: np.ndarray) -> np.ndarray:
    """SynthRng::uniform (form.hpp:751-753): lo + span * double(x) * 0x1.0p-53, same rounding order."""
    return lo + (span * raw) * 2.0 ** -53


def chain_index_map(cells: int, entries: int) -> IndexMap:  # form.hpp:761-768
    overlap = ceil_div(entries, 4)
    stride = entries - overlap
    idx = (np.arange(cells, dtype=np.int64)[:, None] * stride + np.arange(entries)[None, :]).astype(np.int32)
    return IndexMap(idx, (cells - 1) * stride + entries)


def _draw_tabulations(sig: FormSignature, rng: SynthRng) -> Tabulations:
    Q = sig.quad_points
    tab = Tabulations()
    for s in sig.scalar_spaces:
        tab.scalar_phi.append(rng.uniform(0.1, 1.0, s.deriv_terms * Q * s.dofs).reshape(s.deriv_terms, Q, s.dofs))
    for v in sig.vector_spaces:
        tab.vector_phi.append(rng.uniform(0.1, 1.0, v.deriv_terms * Q * v.dofs).reshape(v.deriv_terms, Q, v.dofs))
    tab.psi = rng.uniform(0.1, 1.0, sig.test_deriv_terms * sig.test_dofs * Q).reshape(
        sig.test_deriv_terms, sig.test_dofs, Q)
    tab.weights = rng.uniform(0.5, 0.5, Q)
    return tab


def _seed0(seed: int) -> int:
    return (int(seed) * 0x100000001B3 + 0xCBF29CE484222325) & _MASK64


def make_problem(sig: FormSignature, pmap: PointwiseMap, n_cells: int, seed: int) -> ProblemInstance:
    """form.hpp:774-852 — chain connectivity, near-identity jacobians, positive data."""
    sig.validate()
    if n_cells < 1:
        raise ValueError("make_problem: n_cells >= 1 required")
    rng = SynthRng(_seed0(seed))
    tab = _draw_tabulations(sig, rng)
    conn = MeshConnectivity(cell_count=n_cells)
    conn.scalar_maps = [chain_index_map(n_cells, s.dofs) for s in sig.scalar_spaces]
    conn.vector_maps = [chain_index_map(n_cells, v.dofs) for v in sig.vector_spaces]
    conn.test_map = chain_index_map(n_cells, sig.test_dofs)
    if sig.affine_geometry:
        d, nv = sig.dim, sig.coord_dofs
        conn.coord_map = IndexMap(np.arange(n_cells * nv, dtype=np.int32).reshape(n_cells, nv), n_cells * nv)
        conn.coord_global_count = n_cells * nv
        # per cell, in draw order: base[c] = U(0,1) for c < d, then jitter U(0,0.2) for
        # (j >= 1, c) row-major (form.hpp:826-836)
        per_cell = d + (nv - 1) * d
        raw = rng.raw53(n_cells * per_cell).reshape(n_cells, per_cell)
        base = uniform_from_raw(0.0, 1.0, raw[:, :d])
        jit = uniform_from_raw(0.0, 0.2, raw[:, d:])
        coords = np.empty((n_cells, nv, d))
        coords[:, 0, :] = base
        jit = jit.reshape(n_cells, nv - 1, d)
        for j in range(1, nv):
            for c in range(d):
                v = base[:, c] + jit[:, j - 1, c]
                if c == j - 1:
                    v = v + 1.0
                coords[:, j, c] = v
        conn.coords = coords.reshape(n_cells * nv, d)
    p = ProblemInstance(sig, pmap, tab, conn)
    for m in conn.scalar_maps:
        p.scalar_inputs.append(rng.uniform(0.25, 1.0, m.global_count))
    for m in conn.vector_maps:
        p.vector_inputs.append(rng.uniform(0.25, 1.0, m.global_count * sig.dim))
    p.output_size = conn.test_map.global_count
    p.validate()
    return p


def synthesize_problem(sig: FormSignature, n_cells: int, seed: int) -> ProblemInstance:  # form.hpp:879-881
    return make_problem(sig, generic_map(sig), n_cells, seed)


def fill_inputs(sig: FormSignature, conn: MeshConnectivity, rng: SynthRng):
    """x ~ U[0.25, 1.25) per trial space, same distribution as make_problem (form.hpp:839-848)."""
    xs = [rng.uniform(0.25, 1.0, m.global_count) for m in conn.scalar_maps]
    vs = [rng.uniform(0.25, 1.0, m.global_count * sig.dim) for m in conn.vector_maps]
    return xs, vs
