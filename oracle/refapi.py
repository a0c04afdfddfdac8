"""oracle/refapi.py -- Python access to the CHECKERS (test infrastructure only).

* ``RefSystem``: the reference's own FormSystem, compiled from
  /root/reference/proj/src by oracle/Makefile into oracle/_ref/libtetmf_ref.so
  (see oracle/ref_driver.cpp for the exact reference functions exercised).
* ``PortSystem``: the plain-C restatement in oracle/port/ (oracle/_build/).
* ``seeded_values``: the layout-independent seeded input generator of
  SURVEY.md 8(d), restated in numpy (the product computes the same values on
  the device in k_common.cu; lattice.hpp holds the definition).

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs import this module, and only as the checker / CPU baseline.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libtetmf_ref.so")
REF_FIXED_LIB = os.path.join(HERE, "_ref", "libtetmf_ref_fixed.so")
PORT_LIB = os.path.join(HERE, "_build", "libtetmf_oracle.so")

_dp = ctypes.POINTER(ctypes.c_double)
_ucp = ctypes.POINTER(ctypes.c_ubyte)
_llp = ctypes.POINTER(ctypes.c_longlong)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


# ----------------------------------------------------------------- seeded values
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(z):
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _hash_vertex(X, Y, Z):
    h = _splitmix64(X.astype(np.int64).view(np.uint64) ^ np.uint64(0x5851F42D4C957F2D))
    h = _splitmix64(h ^ Y.astype(np.int64).view(np.uint64))
    return _splitmix64(h ^ Z.astype(np.int64).view(np.uint64))


def _hash_edge(A, B):
    with np.errstate(over="ignore"):
        return _splitmix64(_hash_vertex(*A.T) ^ (_hash_vertex(*B.T) * np.uint64(0x9E3779B97F4A7C15))
                           ^ np.uint64(0xED6E))


def _uniform(seed, h):
    r = _splitmix64(np.uint64(seed) ^ h)
    return 2.0 * ((r >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)) - 1.0


def seeded_values(kind: np.ndarray, a: np.ndarray, b: np.ndarray, scale: int, seed: int,
                  signed_edges: bool = True) -> np.ndarray:
    """Seeded uniform[-1,1] value per DoF from its geometry.

    kind 0: vertex at a; kind 1: edge a -> b (value along a -> b; with
    signed_edges=False -- P2 midpoint DoFs -- the key-ascending edge's value).
    scale: integer such that scale * coordinates are integers (n * D).
    """
    A = np.rint(a * scale).astype(np.int64)
    out = np.empty(len(kind), dtype=np.float64)
    v = kind == 0
    out[v] = _uniform(seed, _hash_vertex(A[v, 0], A[v, 1], A[v, 2]))
    e = ~v
    if e.any():
        B = np.rint(b[e] * scale).astype(np.int64)
        Ae = A[e]
        # lexicographic a < b ?
        less = (Ae[:, 0] < B[:, 0]) | ((Ae[:, 0] == B[:, 0]) & ((Ae[:, 1] < B[:, 1]) |
                                                                ((Ae[:, 1] == B[:, 1]) & (Ae[:, 2] < B[:, 2]))))
        lo = np.where(less[:, None], Ae, B)
        hi = np.where(less[:, None], B, Ae)
        val = _uniform(seed, _hash_edge(lo, hi))
        out[e] = np.where(less, val, -val) if signed_edges else val
    return out


def alpha_fn(p):
    return 1.0 + p[:, 0] ** 2 + p[:, 1] ** 2


def beta_fn(p):
    return 2.0 + np.sin(np.pi * p[:, 2])


def k_fn(p):
    return 1.0 + 0.5 * np.sin(2 * np.pi * p[:, 0]) * np.cos(2 * np.pi * p[:, 1]) * (1.0 + p[:, 2])


# ----------------------------------------------------------------- reference lib
class _Lib:
    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        L = ctypes.CDLL(path)
        p = prefix
        sig = {
            "last_error": (ctypes.c_char_p, []),
            "create": (ctypes.c_void_p, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int]),
            "destroy": (None, [ctypes.c_void_p]),
            "num_dofs": (ctypes.c_longlong, [ctypes.c_void_p]),
            "num_macros": (ctypes.c_int, [ctypes.c_void_p]),
            "dof_geometry": (ctypes.c_int, [ctypes.c_void_p, _ucp, _dp, _dp]),
            "interior": (ctypes.c_int, [ctypes.c_void_p, _ucp]),
            "coeff_num_dofs": (ctypes.c_longlong, [ctypes.c_void_p]),
            "coeff_geometry": (ctypes.c_int, [ctypes.c_void_p, _dp]),
            "interpolate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _dp]),
            "apply": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, ctypes.c_int, _dp, _dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, f"{p}_{name}")
            f.restype = res
            f.argtypes = args
            setattr(self, name, f)
        self.L = L


_REF = None
_PORT = None


def ref_lib():
    global _REF
    if _REF is None:
        _REF = _Lib(REF_LIB, "ref")
        L = _REF.L
        L.ref_local_matrix.restype = ctypes.c_int
        L.ref_local_matrix.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 5 + [_dp, _dp, ctypes.c_int, _dp]
        L.ref_enumerate.restype = ctypes.c_longlong
        L.ref_enumerate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_longlong]
        L.ref_quadrature.restype = ctypes.c_int
        L.ref_quadrature.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_int]
        L.ref_local_dofs.restype = ctypes.c_int
        L.ref_local_dofs.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 5 + [_llp, _dp]
    return _REF


_REF_FIXED = None


def ref_fixed_lib():
    global _REF_FIXED
    if _REF_FIXED is None:
        _REF_FIXED = _Lib(REF_FIXED_LIB, "ref")
        L = _REF_FIXED.L
        L.ref_local_dofs.restype = ctypes.c_int
        L.ref_local_dofs.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 5 + [_llp, _dp]
    return _REF_FIXED


def port_lib():
    global _PORT
    if _PORT is None:
        _PORT = _Lib(PORT_LIB, "port")
    return _PORT


class _System:
    """FormSystem-like handle: mesh name, form ("P1" | "P1K" | "N1"), level."""

    def __init__(self, lib, mesh: str, form: str, level: int):
        self.lib = lib
        self.h = lib.create(mesh.encode(), form.encode(), level)
        if not self.h:
            raise ValueError(lib.last_error().decode())
        self.mesh, self.form, self.level = mesh, form, level

    def __del__(self):
        try:
            if self.h:
                self.lib.destroy(self.h)
        except Exception:
            pass

    @property
    def num_dofs(self) -> int:
        return int(self.lib.num_dofs(self.h))

    def dof_geometry(self):
        n = self.num_dofs
        kind = np.empty(n, dtype=np.uint8)
        a = np.empty((n, 3))
        b = np.empty((n, 3))
        self.lib.dof_geometry(self.h, kind.ctypes.data_as(_ucp), _d(a), _d(b))
        return kind, a, b

    def interior(self):
        out = np.empty(self.num_dofs, dtype=np.uint8)
        self.lib.interior(self.h, out.ctypes.data_as(_ucp))
        return out

    def coeff_geometry(self):
        n = int(self.lib.coeff_num_dofs(self.h))
        a = np.empty((n, 3))
        self.lib.coeff_geometry(self.h, _d(a))
        return a

    def interpolate(self, which: int):
        n = int(self.lib.coeff_num_dofs(self.h))
        out = np.empty(n)
        rc = self.lib.interpolate(self.h, which, _d(out))
        if rc:
            raise ValueError(self.lib.last_error().decode())
        return out

    def apply(self, v, c0=None, c1=None, degree: int = 0):
        """w = A v; degree <= 0: reference_apply rule. Returns (w, seconds)."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        c0 = None if c0 is None else np.ascontiguousarray(c0, dtype=np.float64)
        c1 = None if c1 is None else np.ascontiguousarray(c1, dtype=np.float64)
        w = np.empty(self.num_dofs)
        t = ctypes.c_double()
        rc = self.lib.apply(self.h, _d(v), _d(c0), _d(c1), degree, _d(w), ctypes.byref(t))
        if rc:
            raise ValueError(self.lib.last_error().decode())
        return w, t.value

    def seeded_input(self, seed: int, dirichlet: bool = False, scale: int | None = None):
        kind, a, b = self.dof_geometry()
        s = scale if scale is not None else (1 << self.level)
        x = seeded_values(kind, a, b, s, seed)
        if dirichlet:
            x[self.interior() == 0] = 0.0
        return x

    def coefficients(self):
        """Coefficient fields of the form via the system's own interpolate()."""
        if self.form == "N1":
            return self.interpolate(0), self.interpolate(1)
        if self.form in ("P1K", "P2V"):  # k (P1 for P1K, P2 for P2V: the system's coefficient space)
            return self.interpolate(2), None
        return None, None


class RefSystem(_System):
    """The reference's FormSystem. fixed=True (default): built with the one-line
    DoFIndexer::fill_map cursor fix (oracle/Makefile, DESIGN.md "Reference
    defect"); fixed=False: the verbatim reference, whose apply aliases DoF ids
    at level >= 2 (kept to document the defect)."""

    def __init__(self, mesh, form, level, fixed: bool = True):
        super().__init__(ref_fixed_lib() if fixed else ref_lib(), mesh, form, level)


class PortSystem(_System):
    def __init__(self, mesh, form, level):
        super().__init__(port_lib(), mesh, form, level)


def write_kuhn_mesh(path: str, kx: int, ky: int | None = None, kz: int | None = None):
    """Writes the K^3 Kuhn cube mesh in the reference text format
    (mesh.cpp:143-169), same per-cube rule as cube6 (mesh.cpp:122-141)."""
    ky = kx if ky is None else ky
    kz = kx if kz is None else kz
    verts = [(x, y, z) for z in range(kz + 1) for y in range(ky + 1) for x in range(kx + 1)]

    def vid(x, y, z):
        return x + (kx + 1) * (y + (ky + 1) * z)

    tets = []
    perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    for cz in range(kz):
        for cy in range(ky):
            for cx in range(kx):
                for p in perms:
                    a = [0, 0, 0]
                    a[p[0]] = 1
                    b = list(a)
                    b[p[1]] = 1
                    t = [vid(cx, cy, cz), vid(cx + a[0], cy + a[1], cz + a[2]),
                         vid(cx + b[0], cy + b[1], cz + b[2]), vid(cx + 1, cy + 1, cz + 1)]
                    P = np.array([verts[i] for i in t], dtype=float)
                    if np.linalg.det((P[1:] - P[0]).T) < 0:
                        t[2], t[3] = t[3], t[2]
                    tets.append(t)
    with open(path, "w") as f:
        for v in verts:
            f.write(f"v {v[0]} {v[1]} {v[2]}\n")
        for t in tets:
            f.write(f"t {t[0]} {t[1]} {t[2]} {t[3]}\n")
    return path
