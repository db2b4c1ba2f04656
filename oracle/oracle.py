"""TEST INFRASTRUCTURE — ctypes front-end of the C restatement oracle (klref_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use this,
as the checker; the product path never imports it.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None
PROBLEMS = {"zero": 0, "sin": 1, "lshape": 2}


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise ImportError("oracle/liboracle.so missing: make -C oracle")
        L = C.CDLL(path)
        P, I, D = C.c_void_p, C.c_int, C.c_double
        PD, PI = C.POINTER(C.c_double), C.POINTER(C.c_int)
        PPD = C.POINTER(PD)
        sig = {
            "o2_build": (P, [I, PD, I, PI, I]),
            "o2_free": (None, [P]),
            "o2_num_macros": (I, [P]),
            "o2_level_size": (I, [P, I]),
            "o2_dofs": (C.c_longlong, [P, I]),
            "o2_interface_sync": (None, [P, I, PD, I]),
            "o2_dot_unique": (D, [P, I, PD, PD]),
            "o2_apply": (None, [P, I, I, PD, PD]),
            "o2_residual": (None, [P, I, PD, PD, PD]),
            "o2_gauss_seidel": (None, [P, I, PD, PD, I]),
            "o2_prolongate": (None, [P, I, PD, PD]),
            "o2_restrict": (None, [P, I, PD, PD]),
            "o2_cg_level0": (I, [P, PD, PD, D, D, I, PI]),
            "o2_fmg": (I, [P, I, I, I, I, D, D, I, PPD, PPD, PPD]),
            "o2_estimate": (I, [P, PD, PPD, I, I, PD, PD]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Hier2D:
    """Oracle hierarchy (restates GridHierarchy::build, proj/src/hhg.cpp:48-144)."""

    def __init__(self, mesh, L):
        xy = np.ascontiguousarray(mesh.coords[:, :2], dtype=np.float64)
        tri = np.ascontiguousarray(mesh.elements, dtype=np.int32)
        self.ptr = lib().o2_build(xy.shape[0], _pd(xy), tri.shape[0], tri.ctypes.data_as(C.POINTER(C.c_int)), L)
        if not self.ptr:
            raise ValueError("oracle: invalid mesh / level")
        self.L = L
        self.M = tri.shape[0]

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().o2_free(self.ptr)
            self.ptr = None

    def size(self, l):
        return lib().o2_level_size(self.ptr, l)

    def dofs(self, l):
        return lib().o2_dofs(self.ptr, l)

    def apply(self, l, x, mass=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        lib().o2_apply(self.ptr, l, int(mass), _pd(x), _pd(y))
        return y

    def residual(self, l, u, b):
        u = np.ascontiguousarray(u, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        r = np.empty_like(u)
        lib().o2_residual(self.ptr, l, _pd(u), _pd(b), _pd(r))
        return r

    def gauss_seidel(self, l, u, b, sweeps):
        u = np.array(u, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        lib().o2_gauss_seidel(self.ptr, l, _pd(u), _pd(b), sweeps)
        return u

    def prolongate(self, lc, c):
        c = np.ascontiguousarray(c, dtype=np.float64)
        f = np.empty(self.size(lc + 1))
        lib().o2_prolongate(self.ptr, lc, _pd(c), _pd(f))
        return f

    def restrict(self, lf, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        c = np.empty(self.size(lf - 1))
        lib().o2_restrict(self.ptr, lf, _pd(f), _pd(c))
        return c

    def cg_level0(self, u, b, rel=1e-9, absf=1e-12, maxit=100000):
        u = np.array(u, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        it = C.c_int()
        st = lib().o2_cg_level0(self.ptr, _pd(u), _pd(b), rel, absf, maxit, C.byref(it))
        return u, st, it.value

    def dot_unique(self, l, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return lib().o2_dot_unique(self.ptr, l, _pd(a), _pd(b))

    def interface_sync(self, l, f, additive):
        f = np.array(f, dtype=np.float64)
        lib().o2_interface_sync(self.ptr, l, _pd(f), int(additive))
        return f


def fmg2d(mesh, L, problem="sin", nu=2, pre=2, post=2, rel=1e-9, absf=1e-12, maxit=100000, hier=None):
    """MultigridSolver::fmg (FinestPolicy::None) restated; returns u, b, w lists."""
    h = hier or Hier2D(mesh, L)
    u = [np.zeros(h.size(l)) for l in range(L + 1)]
    b = [np.zeros(h.size(l)) for l in range(L + 1)]
    w = [np.zeros(h.size(l + 1)) for l in range(L)]
    PPD = C.POINTER(C.c_double) * (L + 1)
    up = PPD(*[_pd(a) for a in u])
    bp = PPD(*[_pd(a) for a in b])
    wp = PPD(*([_pd(a) for a in w] + [None]))
    st = lib().o2_fmg(h.ptr, PROBLEMS[problem], nu, pre, post, rel, absf, maxit, up, bp, wp)
    return {"u": u, "b": b, "w": w, "status": st, "hier": h, "L": L}


def estimate2d(state, offset=1, kind=0):
    """error_estimate restated (proj/src/estimator.cpp:8-45)."""
    h = state["hier"]
    L = state["L"]
    out = np.zeros(4)
    loc = np.zeros(h.M)
    PPD = C.POINTER(C.c_double) * L
    wp = PPD(*[_pd(a) for a in state["w"]])
    uL = np.ascontiguousarray(state["u"][L])
    rc = lib().o2_estimate(h.ptr, _pd(uL), wp, offset, kind, _pd(out), _pd(loc))
    if rc:
        raise ValueError("estimate offset must satisfy 1 <= j <= L-1")
    return {"norm_base": out[0], "norm_coarser": out[1], "conv": out[2], "eta": out[3], "eta_local": loc}


# ---------------------------------------------------------------- 3-d (configs 3-5)
# The reference has no 3-d solver: klref_oracle3d.c restates the builder's 3-d
# specification (parity unpinned against the reference).
PROBLEMS3D = {"zero": 0, "sin3": 1, "gauss": 2, "series": 3}
_lib3 = None


def lib3():
    global _lib3
    if _lib3 is None:
        L = lib()
        P, I, D = C.c_void_p, C.c_int, C.c_double
        PD, PI = C.POINTER(C.c_double), C.POINTER(C.c_int)
        PPD = C.POINTER(PD)
        sig = {
            "o3_build": (P, [I, PD, I, PI, I]),
            "o3_free": (None, [P]),
            "o3_num_macros": (I, [P]),
            "o3_level_size": (I, [P, I]),
            "o3_dofs": (C.c_longlong, [P, I]),
            "o3_colors": (I, [P]),
            "o3_apply": (None, [P, I, I, PD, PD]),
            "o3_residual": (None, [P, I, PD, PD, PD]),
            "o3_gauss_seidel": (None, [P, I, PD, PD, I]),
            "o3_prolongate": (None, [P, I, PD, PD]),
            "o3_restrict": (None, [P, I, PD, PD]),
            "o3_dot": (D, [P, I, PD, PD]),
            "o3_rhs": (None, [P, I, I, PD, PD]),
            "o3_cg0": (I, [P, PD, PD, D, D, I, PI]),
            "o3_fmg": (I, [P, I, PD, I, I, I, D, D, I, PPD, PPD, PPD]),
            "o3_estimate": (I, [P, PD, PPD, PD, PD]),
            "o3_coords": (None, [P, I, PD]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib3 = L
    return _lib3


class Hier3D:
    """3-d oracle hierarchy: tet lattices, barycentric-key groups, colouring."""

    def __init__(self, coords, tets, L):
        xyz = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(tets, dtype=np.int32).reshape(-1, 4)
        self.ptr = lib3().o3_build(xyz.shape[0], _pd(xyz), t.shape[0], t.ctypes.data_as(C.POINTER(C.c_int)), L)
        if not self.ptr:
            raise ValueError("oracle: invalid 3-d mesh / level")
        self.L = L
        self.M = t.shape[0]

    def __del__(self):
        if getattr(self, "ptr", None):
            lib3().o3_free(self.ptr)
            self.ptr = None

    def size(self, l):
        return lib3().o3_level_size(self.ptr, l)

    def dofs(self, l):
        return lib3().o3_dofs(self.ptr, l)

    def colors(self):
        return lib3().o3_colors(self.ptr)

    def apply(self, l, x, mass=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        lib3().o3_apply(self.ptr, l, int(mass), _pd(x), _pd(y))
        return y

    def residual(self, l, u, b):
        u = np.ascontiguousarray(u, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        r = np.empty_like(u)
        lib3().o3_residual(self.ptr, l, _pd(u), _pd(b), _pd(r))
        return r

    def gauss_seidel(self, l, u, b, sweeps):
        u = np.array(u, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        lib3().o3_gauss_seidel(self.ptr, l, _pd(u), _pd(b), sweeps)
        return u

    def prolongate(self, lc, c):
        c = np.ascontiguousarray(c, dtype=np.float64)
        f = np.empty(self.size(lc + 1))
        lib3().o3_prolongate(self.ptr, lc, _pd(c), _pd(f))
        return f

    def restrict(self, lf, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        c = np.empty(self.size(lf - 1))
        lib3().o3_restrict(self.ptr, lf, _pd(f), _pd(c))
        return c

    def dot(self, l, a, b):
        return lib3().o3_dot(self.ptr, l, _pd(np.ascontiguousarray(a)), _pd(np.ascontiguousarray(b)))

    def coords(self, l):
        out = np.empty((self.size(l), 3))
        lib3().o3_coords(self.ptr, l, _pd(out))
        return out


def fmg3d(hier, problem="sin3", params=None, nu=2, pre=2, post=2, rel=1e-9, absf=1e-12, maxit=100000):
    h = hier
    L = h.L
    par = np.zeros(64) if params is None else np.ascontiguousarray(params, dtype=np.float64)
    u = [np.zeros(h.size(l)) for l in range(L + 1)]
    b = [np.zeros(h.size(l)) for l in range(L + 1)]
    w = [np.zeros(h.size(l + 1)) for l in range(L)]
    PPD = C.POINTER(C.c_double) * (L + 1)
    up = PPD(*[_pd(a) for a in u])
    bp = PPD(*[_pd(a) for a in b])
    wp = PPD(*([_pd(a) for a in w] + [None]))
    st = lib3().o3_fmg(h.ptr, PROBLEMS3D[problem], _pd(par), nu, pre, post, rel, absf, maxit, up, bp, wp)
    return {"u": u, "b": b, "w": w, "status": st, "hier": h, "L": L}


def estimate3d(state):
    h = state["hier"]
    L = state["L"]
    out = np.zeros(4)
    loc = np.zeros(2 * h.M)
    PPD = C.POINTER(C.c_double) * L
    wp = PPD(*[_pd(a) for a in state["w"]])
    uL = np.ascontiguousarray(state["u"][L])
    if lib3().o3_estimate(h.ptr, _pd(uL), wp, _pd(out), _pd(loc)):
        raise ValueError("3-d estimate needs L >= 2")
    return {"norm_base": out[0], "norm_coarser": out[1], "conv": out[2], "eta": out[3],
            "local_base": np.sqrt(np.maximum(loc[0::2], 0.0)), "local_sums": loc}
