"""Reference-element tables of the nodal tensor-product DG basis.

Same conventions as the reference (orodg/basis.py:1-12, 157-207): solution
nodes are the Gauss-Lobatto-Legendre points on [0, 1], quadrature is
Gauss-Legendre with n_q points per axis (n_q = r + 1 by default), node and
quadrature flattening is C-order over (x, y, z) with z fastest.

Only 1D tables matter on the device: the sum-factorised kernels apply the
1D matrices axis by axis.  The dense Kronecker operators are kept as lazily
built host conveniences for the CPU oracle and the API surface.

Derived 1D tables used by the B200 kernels:
  * ``Binv``  = B^-1 (B = interp_1d is square when n_q = r+1),
  * ``Dhat``  = D B^-1, the collocation derivative at Gauss points,
  * ``lift``  = B^-T e_{0}, B^-T e_{r}: a nodal trace/lift expressed on the
    Gauss points of the normal axis,
  * ``half_q`` = half_interp_1d[s] B^-1: mortar half interpolation acting on
    Gauss-point traces.
"""

import functools
from dataclasses import dataclass, field

import numpy as np


def gauss_legendre(n):
    """Gauss-Legendre points and weights mapped to [0, 1]."""
    t, w = np.polynomial.legendre.leggauss(n)
    return (t + 1.0) * 0.5, w * 0.5


def gauss_lobatto(n):
    """Gauss-Lobatto-Legendre points on [0, 1]: the endpoints plus the roots
    of P'_{n-1}."""
    if n < 2:
        raise ValueError("GLL rule needs at least 2 nodes")
    if n == 2:
        return np.array([0.0, 1.0])
    c = np.zeros(n)
    c[n - 1] = 1.0
    inner = np.polynomial.legendre.legroots(np.polynomial.legendre.legder(c))
    return (np.concatenate(([-1.0], inner, [1.0])) + 1.0) * 0.5


def _bary_weights(x):
    n = len(x)
    w = np.ones(n)
    for j in range(n):
        for k in range(n):
            if k != j:
                w[j] /= (x[j] - x[k])
    return w


def lagrange_eval_matrix(nodes, points):
    """L[p, j] = l_j(points[p]) (second barycentric form; rows that hit a
    node exactly are the exact unit rows, which keeps shared face surfaces
    bitwise identical from both sides)."""
    x = np.asarray(nodes, dtype=float)
    p = np.atleast_1d(np.asarray(points, dtype=float))
    w = _bary_weights(x)
    out = np.empty((len(p), len(x)))
    for i, pt in enumerate(p):
        dist = pt - x
        hit = np.nonzero(np.abs(dist) <= 1e-14)[0]
        if len(hit):
            out[i] = 0.0
            out[i, hit[0]] = 1.0
            continue
        t = w / dist
        out[i] = t / t.sum()
    return out


def lagrange_diff_matrix(nodes, points):
    """D[p, j] = l_j'(points[p]) from the product rule,
    l_j' = sum_m prod_{k != j, m} (x - x_k) / prod_{k != j} (x_j - x_k)."""
    x = np.asarray(nodes, dtype=float)
    p = np.atleast_1d(np.asarray(points, dtype=float))
    n = len(x)
    out = np.zeros((len(p), n))
    for j in range(n):
        others = [k for k in range(n) if k != j]
        den = np.prod([x[j] - x[k] for k in others])
        acc = np.zeros(len(p))
        for m in others:
            term = np.ones(len(p))
            for k in others:
                if k != m:
                    term = term * (p - x[k])
            acc += term
        out[:, j] = acc / den
    return out


def _kron(mats):
    out = mats[0]
    for m in mats[1:]:
        out = np.kron(out, m)
    return out


def _face_nodes(dim, n1):
    grid = np.arange(n1 ** dim).reshape((n1,) * dim)
    res = []
    for axis in range(dim):
        lo = np.take(grid, 0, axis=axis).ravel()
        hi = np.take(grid, n1 - 1, axis=axis).ravel()
        res.append((lo, hi))
    return tuple(res)


@dataclass(frozen=True)
class ReferenceBasis:
    """Degree-r nodal tensor basis with Gauss quadrature (orodg/basis.py:95-139)."""

    dim: int
    degree: int
    n_quad_1d: int
    nodes_1d: np.ndarray
    quad_x: np.ndarray
    quad_w: np.ndarray
    interp_1d: np.ndarray
    diff_1d: np.ndarray
    trace_1d: np.ndarray
    half_interp_1d: tuple
    face_nodes: tuple
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    # -- sizes --------------------------------------------------------------
    @property
    def n_nodes(self):
        return (self.degree + 1) ** self.dim

    @property
    def n_quad(self):
        return self.n_quad_1d ** self.dim

    @property
    def n_face_nodes(self):
        return (self.degree + 1) ** (self.dim - 1)

    @property
    def n_face_quad(self):
        return self.n_quad_1d ** (self.dim - 1)

    @property
    def n_subfaces(self):
        return 2 ** (self.dim - 1)

    def subface_coords(self, subface):
        return tuple((subface >> i) & 1 for i in range(self.dim - 1))

    # -- dense Kronecker operators (host conveniences) ----------------------
    def _memo(self, key, fn):
        if key not in self._cache:
            self._cache[key] = fn()
        return self._cache[key]

    @property
    def vol_interp(self):
        return self._memo("vi", lambda: _kron([self.interp_1d] * self.dim))

    @property
    def vol_diff(self):
        def build():
            out = []
            for a in range(self.dim):
                mats = [self.interp_1d] * self.dim
                mats[a] = self.diff_1d
                out.append(_kron(mats))
            return tuple(out)
        return self._memo("vd", build)

    @property
    def vol_w(self):
        return self._memo("vw", lambda: _kron([self.quad_w[None, :]] * self.dim).ravel())

    @property
    def face_interp(self):
        return self._memo("fi", lambda: _kron([self.interp_1d] * (self.dim - 1)))

    @property
    def face_w(self):
        return self._memo("fw", lambda: _kron([self.quad_w[None, :]] * (self.dim - 1)).ravel())

    @property
    def mortar_interp(self):
        def build():
            return tuple(_kron([self.half_interp_1d[(s >> i) & 1]
                                for i in range(self.dim - 1)])
                         for s in range(self.n_subfaces))
        return self._memo("mi", build)

    # -- derived 1D tables for the sum-factorised device kernels ------------
    @property
    def square(self):
        return self.n_quad_1d == self.degree + 1

    @property
    def Binv(self):
        return self._memo("binv", lambda: np.linalg.inv(self.interp_1d))

    @property
    def Dhat(self):
        return self._memo("dhat", lambda: self.diff_1d @ self.Binv)

    @property
    def lift(self):
        """(2, n_q): row s = B^-T e_{end_s}; trace of a Gauss-point column is
        lift[s] . column, and a nodal face lift is lift[s] (x) face values."""
        return self._memo("lift", lambda: np.ascontiguousarray(
            self.Binv[[0, self.degree], :]))

    @property
    def half_q(self):
        return self._memo("halfq", lambda: tuple(h @ self.Binv for h in self.half_interp_1d))


@functools.lru_cache(maxsize=None)
def make_basis(dim, degree, n_quad_1d=None):
    """Build the basis tables (orodg/basis.py:157-207)."""
    if dim not in (2, 3):
        raise ValueError("dim must be 2 or 3")
    if degree < 1:
        raise ValueError("degree must be >= 1")
    nq = degree + 1 if n_quad_1d is None else int(n_quad_1d)
    x = gauss_lobatto(degree + 1)
    qx, qw = gauss_legendre(nq)
    B = lagrange_eval_matrix(x, qx)
    D = lagrange_diff_matrix(x, qx)
    tr = lagrange_eval_matrix(x, np.array([0.0, 1.0]))
    half = tuple(lagrange_eval_matrix(x, 0.5 * (qx + s)) for s in (0, 1))
    return ReferenceBasis(dim=dim, degree=degree, n_quad_1d=nq, nodes_1d=x,
                          quad_x=qx, quad_w=qw, interp_1d=B, diff_1d=D,
                          trace_1d=tr, half_interp_1d=half,
                          face_nodes=_face_nodes(dim, degree + 1))
