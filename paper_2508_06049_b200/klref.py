"""Python mirror of the reference's hot-path API over the C-ABI of libklref_b200.so.

The names follow the reference's C++ interface (proj/include/klref/*.hpp):
``GridHierarchy.build`` (hhg.hpp:78), ``MultigridSolver`` / ``fmg`` /
``gauss_seidel`` / ``residual`` / ``cg_level0`` (multigrid.hpp:64-99),
``OperatorP1.apply`` (fem.hpp:26-40), ``restrict_transpose`` / ``prolongate``
(multigrid.hpp:56-60), ``dot_unique`` / ``interface_sync`` (hhg.hpp:134-137),
``error_estimate`` (estimator.hpp:26).  Errors raise the Python counterparts of
proj/include/klref/errors.hpp.  Every compute call runs the sm_100a kernels;
there is no CPU fallback (a missing library or device raises).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KLREF_LIB") or os.path.join(_HERE, "libklref_b200.so")


# ---------------------------------------------------------------- errors
class KlrefError(RuntimeError):
    code = -1


class StructuralError(KlrefError):
    code = 1


class DomainError(KlrefError):
    code = 2


class SolverError(KlrefError):
    code = 3

    def __init__(self, msg, last_residual=0.0):
        super().__init__(msg)
        self.last_residual = last_residual


class IoError(KlrefError):
    code = 4


class InternalError(KlrefError):
    code = 5


class ResourceError(KlrefError):
    code = 6

    def __init__(self, msg, level=-1):
        super().__init__(msg)
        self.level = level


class CudaError(KlrefError):
    code = 7


_ERRORS = {1: StructuralError, 2: DomainError, 3: SolverError, 4: IoError, 5: InternalError,
           6: ResourceError, 7: CudaError}

STIFFNESS, MASS = 0, 1
UNSCALED, SCALED = 0, 1
SYNC_REPLACE, SYNC_ADDITIVE = 0, 1
STATE_U, STATE_B, STATE_W = 0, 1, 2
PROBLEM_ZERO, PROBLEM_SIN2D, PROBLEM_LSHAPE = 0, 1, 2
POLICY_NONE, POLICY_VALIDATION_TWO_DIGITS, POLICY_RESIDUAL_VS_ESTIMATE = 0, 1, 2
PROBLEM_SIN3D, PROBLEM_GAUSS3D, PROBLEM_SERIES3D = 3, 4, 5
MARK_TOP_FRACTION, MARK_HALF_MAX = 0, 1
KERNEL_ALL, KERNEL_GS, KERNEL_RESIDUAL, KERNEL_RESTRICT, KERNEL_PROLONG = -1, 0, 1, 2, 3
KERNEL_RHS, KERNEL_CG0, KERNEL_ESTIMATE, KERNEL_OTHER = 4, 5, 6, 7
KERNEL_NAMES = {0: "gauss_seidel", 1: "residual", 2: "restrict", 3: "prolongate", 4: "rhs", 5: "cg_level0",
                6: "estimate", 7: "other"}


class SolverConfigC(C.Structure):
    _fields_ = [("nu", C.c_int), ("pre_smooth", C.c_int), ("post_smooth", C.c_int),
                ("coarse_rel_tol", C.c_double), ("coarse_abs_floor", C.c_double),
                ("coarse_max_iter", C.c_int), ("finest_policy", C.c_int),
                ("faithful_source", C.c_int), ("use_graph", C.c_int), ("max_extra_cycles", C.c_int)]


class EstimateReportC(C.Structure):
    _fields_ = [("offset", C.c_int), ("base_level", C.c_int), ("kind", C.c_int),
                ("norm_coarser", C.c_double), ("norm_base", C.c_double),
                ("conv_factor", C.c_double), ("eta", C.c_double)]


_lib = None

# exported symbols and their ctypes signatures (include/klref_b200.h)
_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_PI = C.POINTER(C.c_int)
_PD = C.POINTER(C.c_double)
_PP = C.POINTER(C.c_void_p)
_PI64 = C.POINTER(C.c_int64)
SIGNATURES = {
    "klref_last_error": (C.c_char_p, []),
    "klref_last_error_residual": (_D, []),
    "klref_last_error_level": (_I, []),
    "klref_device_init": (_I, []),
    "klref_abi_version": (_I, []),
    "klref_mesh_create": (_I, [_I, _I, _PD, _I, _PI, _PP]),
    "klref_mesh_destroy": (None, [_P]),
    "klref_hierarchy_build": (_I, [_P, _I, _PP]),
    "klref_hierarchy_build_host": (_I, [_P, _I, _PP]),
    "klref_hierarchy_destroy": (None, [_P]),
    "klref_hierarchy_num_macros": (_I, [_P, _PI]),
    "klref_hierarchy_max_level": (_I, [_P, _PI]),
    "klref_hierarchy_dof_count": (_I, [_P, _I, _PI64]),
    "klref_hierarchy_fine_element_count": (_I, [_P, _I, _PI64]),
    "klref_hierarchy_lattice_size": (_I, [_P, _I, _PI]),
    "klref_hierarchy_dag_depth": (_I, [_P, _PI]),
    "klref_hierarchy_groups": (_I, [_P, _I, _PI, _PI, _PI, _PI]),
    "klref_hierarchy_element_matrices": (_I, [_P, _I, _I, _PD, _PD]),
    "klref_problem_create": (_I, [_I, _PP]),
    "klref_problem_create_host": (_I, [_P, _P, _P, _PP]),
    "klref_problem_create_host3": (_I, [_P, _P, _P, _PP]),
    "klref_problem_set_params": (_I, [_P, _PD, _I]),
    "klref_problem_set_exact": (_I, [_P, _P, _P]),
    "klref_solver_exact_error": (_I, [_P, _PD, _PD]),
    "klref_solver_exact_error_of": (_I, [_P, _P, _PD, _PD]),
    "klref_solver_solve_direct": (_I, [_P, _I, _P]),
    "klref_solver_extra_cycles": (_I, [_P, _PI]),
    "klref_problem_destroy": (None, [_P]),
    "klref_solver_config_default": (None, [C.POINTER(SolverConfigC)]),
    "klref_solver_create": (_I, [_P, _P, C.POINTER(SolverConfigC), _PP]),
    "klref_solver_destroy": (None, [_P]),
    "klref_solver_fmg": (_I, [_P]),
    "klref_solver_fmg_enqueue": (_I, [_P]),
    "klref_solver_synchronize": (_I, [_P]),
    "klref_solver_stream": (_I, [_P, _PP]),
    "klref_solver_launch_count": (_I, [_P, _PI]),
    "klref_solver_last_cg_iterations": (_I, [_P, _PI]),
    "klref_solver_state_read": (_I, [_P, _I, _I, _PD]),
    "klref_solver_estimate_launch_count": (_I, [_P, _PI]),
    "klref_solver_set_stream": (_I, [_P, _P]),
    "klref_solver_set_problem": (_I, [_P, _P, _PI64]),
    "klref_solver_set_profiling": (_I, [_P, _I]),
    "klref_solver_kernel_stats": (_I, [_P, _I, _PD, _PI, _PD]),
    "klref_error_estimate": (_I, [_P, _I, _I, C.POINTER(EstimateReportC), _PD]),
    "klref_error_estimate_enqueue": (_I, [_P, _I]),
    "klref_error_estimate_finish": (_I, [_P, _I, _I, C.POINTER(EstimateReportC), _PD]),
    "klref_gf_create": (_I, [_P, _I, _PP]),
    "klref_gf_destroy": (None, [_P]),
    "klref_gf_upload": (_I, [_P, _PD]),
    "klref_gf_download": (_I, [_P, _PD]),
    "klref_apply": (_I, [_P, _I, _P, _P]),
    "klref_residual": (_I, [_P, _P, _P, _P]),
    "klref_gauss_seidel": (_I, [_P, _P, _P, _I]),
    "klref_restrict_transpose": (_I, [_P, _P, _P]),
    "klref_prolongate": (_I, [_P, _P, _P]),
    "klref_cg_level0": (_I, [_P, _P, _P]),
    "klref_dot_unique": (_I, [_P, _P, _P, _PD]),
    "klref_interface_sync": (_I, [_P, _P, _I]),
    "klref_mark": (_I, [_I, _D, _I, _PI, _PI, _PD, _I, _PI, _PI, _PI]),
    "klref_effectivity_constants": (_I, [_D, _D, _I, _PD, _PD]),
    "klref_local_spread_bound_scaled": (_I, [_D, _D, _I, _PD]),
    "klref_local_spread_bound_unscaled": (_I, [_D, _D, _I, _PD]),
    "klref_effectivity_index": (_I, [_D, _I, _PD, _D, _I, _PD, _PD, _PI, _PD, _PD, _PI]),
    "klref_comm_unique_id": (_I, [C.c_char_p]),
    "klref_comm_create": (_I, [_I, _I, C.c_char_p, _PP]),
    "klref_comm_destroy": (None, [_P]),
    "klref_sharded_create": (_I, [_P, _P, C.POINTER(SolverConfigC), _P, _I, _I, _PP]),
    "klref_sharded_destroy": (None, [_P]),
    "klref_sharded_fmg": (_I, [_P]),
    "klref_sharded_fmg_enqueue": (_I, [_P]),
    "klref_sharded_synchronize": (_I, [_P]),
    "klref_sharded_stream": (_I, [_P, _PP]),
    "klref_sharded_counts": (_I, [_P, _PI, _PI, _PD]),
    "klref_sharded_error_estimate_enqueue": (_I, [_P, _I]),
    "klref_sharded_error_estimate_finish": (_I, [_P, _I, _I, C.POINTER(EstimateReportC), _PD]),
    "klref_sharded_state_read": (_I, [_P, _I, _I, _PD]),
    "klref_shard_starts": (_I, [_I, _I, _PI]),
    "klref_shard_plan": (_I, [_P, _I, _I, _I, _I, _PI, _PI64, _PI64, _PI, _PI]),
}


def lib():
    """Load libklref_b200.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() (make -C csrc)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    L = lib()
    msg = L.klref_last_error().decode()
    cls = _ERRORS.get(rc, KlrefError)
    if cls is SolverError:
        raise SolverError(msg, L.klref_last_error_residual())
    if cls is ResourceError:
        raise ResourceError(msg, L.klref_last_error_level())
    raise cls(msg)


def _dptr(a: np.ndarray):
    # the C side reads / writes count contiguous doubles from this address
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise ValueError("expected a C-contiguous float64 array")
    return a.ctypes.data_as(_PD)


def _iptr(a: np.ndarray):
    if a.dtype != np.int32 or not a.flags.c_contiguous:
        raise ValueError("expected a C-contiguous int32 array")
    return a.ctypes.data_as(_PI)


# ---------------------------------------------------------------- lattice helpers
def lattice_index(n: int, i: int, j: int) -> int:
    """proj/include/klref/hhg.hpp:13"""
    return j * (n + 1) - (j * (j - 1)) // 2 + i


def lattice_size(n: int) -> int:
    return (n + 1) * (n + 2) // 2


# ---------------------------------------------------------------- mesh
@dataclass
class MacroMesh:
    """Active conforming macro mesh: coords[nv, 2], elements[ne, 3] (slot order)."""
    coords: np.ndarray
    elements: np.ndarray
    dim: int = 2

    @staticmethod
    def read(path: str) -> "MacroMesh":
        """ASCII format of proj/include/klref/mesh_io.hpp:14-22 (read_mesh, mesh_io.cpp:31-96)."""
        lines = []
        with open(path) as fh:
            for ln in fh:
                s = ln.strip()
                if s and not s.startswith("#"):
                    lines.append(s)
        it = iter(lines)
        tag, dim = next(it).split()
        if tag != "dim":
            raise IoError("expected 'dim d' header")
        dim = int(dim)
        tag, nv = next(it).split()
        nv = int(nv)
        ids, coords = [], []
        for _ in range(nv):
            parts = next(it).split()
            ids.append(int(parts[0]))
            coords.append([float(v) for v in parts[1:1 + dim]])
        idmap = {v: k for k, v in enumerate(ids)}
        tag, ne = next(it).split()
        elements = []
        for _ in range(int(ne)):
            parts = next(it).split()
            elements.append([idmap[int(v)] for v in parts[1:2 + dim]])
        return MacroMesh(np.array(coords, dtype=np.float64), np.array(elements, dtype=np.int32), dim)

    def boundary_vertices(self) -> np.ndarray:
        """Per vertex: on the domain boundary (a facet used by exactly one element),
        the flag column of the mesh format (proj/src/mesh_io.cpp:121-127)."""
        from collections import Counter
        d = self.dim
        cnt = Counter()
        for el in self.elements:
            for skip in range(d + 1):
                cnt[tuple(sorted(int(v) for t, v in enumerate(el) if t != skip))] += 1
        flag = np.zeros(len(self.coords), dtype=bool)
        for facet, c in cnt.items():
            if c == 1:
                flag[list(facet)] = True
        return flag

    def write(self, path: str) -> None:
        """write_mesh of the reference (proj/src/mesh_io.cpp:104-143): header, the
        referenced vertices renumbered compactly in ascending id order with %.17g
        coordinates and the boundary flag, the elements in slot order."""
        used = sorted({int(v) for el in self.elements for v in el})
        new = {old: k for k, old in enumerate(used)}
        bnd = self.boundary_vertices()
        with open(path, "w") as fh:
            fh.write("# written " + time.strftime("%Y-%m-%d %H:%M:%S", time.gmtime()) + " UTC\n")
            fh.write(f"dim {self.dim}\n")
            fh.write(f"vertices {len(used)}\n")
            for old in used:
                xs = " ".join("%.17g" % float(c) for c in self.coords[old][: self.dim])
                fh.write(f"{new[old]} {xs} {1 if bnd[old] else 0}\n")
            fh.write(f"elements {len(self.elements)}\n")
            for e, el in enumerate(self.elements):
                fh.write(str(e) + " " + " ".join(str(new[int(v)]) for v in el) + "\n")


def write_marks(path: str, ids) -> None:
    """Marks file in the format read_marks_file accepts (proj/src/mesh_io.cpp:145-163):
    element positions of the written mesh, whitespace separated, '#' comments."""
    with open(path, "w") as fh:
        fh.write("# marked elements (positions in the mesh file)\n")
        fh.write(" ".join(str(int(i)) for i in sorted(set(int(i) for i in ids))) + "\n")


def read_marks(path: str, num_elements: int) -> np.ndarray:
    """read_marks_file (proj/src/mesh_io.cpp:145-163): sorted unique ids, range-checked."""
    ids = []
    try:
        fh = open(path)
    except OSError as e:
        raise IoError(f"cannot open marks file: {path}") from e
    with fh:
        for ln in fh:
            ln = ln.split("#", 1)[0]
            for tok in ln.split():
                v = int(tok)
                if v < 0 or v >= num_elements:
                    raise IoError(f"mark id out of range: {v}")
                ids.append(v)
    return np.array(sorted(set(ids)), dtype=np.int64)


class _Handle:
    _destroy = None

    def __init__(self, ptr):
        self._ptr = ptr

    @property
    def ptr(self):
        return self._ptr

    def close(self):
        if self._ptr:
            getattr(lib(), self._destroy)(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Mesh(_Handle):
    _destroy = "klref_mesh_destroy"

    def __init__(self, mm: MacroMesh):
        out = C.c_void_p()
        coords = np.ascontiguousarray(mm.coords, dtype=np.float64)
        els = np.ascontiguousarray(mm.elements, dtype=np.int32)
        _check(lib().klref_mesh_create(mm.dim, coords.shape[0], _dptr(coords), els.shape[0], _iptr(els),
                                       C.byref(out)))
        super().__init__(out.value)
        self.macro = mm


class GridHierarchy(_Handle):
    """GridHierarchy (proj/include/klref/hhg.hpp:56-128), device resident."""
    _destroy = "klref_hierarchy_destroy"

    @staticmethod
    def build(mesh: MacroMesh, max_level: int, device: bool = True) -> "GridHierarchy":
        m = Mesh(mesh)
        out = C.c_void_p()
        fn = lib().klref_hierarchy_build if device else lib().klref_hierarchy_build_host
        _check(fn(m.ptr, max_level, C.byref(out)))
        h = GridHierarchy(out.value)
        h.mesh = m
        h.dim = int(mesh.dim)
        return h

    def _int(self, fn, *args):
        v = C.c_int()
        _check(fn(self.ptr, *args, C.byref(v)))
        return v.value

    def _i64(self, fn, *args):
        v = C.c_int64()
        _check(fn(self.ptr, *args, C.byref(v)))
        return v.value

    def num_macros(self):
        return self._int(lib().klref_hierarchy_num_macros)

    def max_level(self):
        return self._int(lib().klref_hierarchy_max_level)

    def dof_count(self, l):
        return self._i64(lib().klref_hierarchy_dof_count, l)

    def fine_element_count(self, l):
        return self._i64(lib().klref_hierarchy_fine_element_count, l)

    def lattice_size(self, l):
        return self._int(lib().klref_hierarchy_lattice_size, l)

    def level_size(self, l):
        return self.num_macros() * self.lattice_size(l)

    def dag_depth(self):
        return self._int(lib().klref_hierarchy_dag_depth)

    def groups(self, l):
        ng, nm = C.c_int(), C.c_int()
        _check(lib().klref_hierarchy_groups(self.ptr, l, C.byref(ng), C.byref(nm), None, None))
        ptr = np.zeros(ng.value + 1, dtype=np.int32)
        mem = np.zeros((nm.value, 4), dtype=np.int32)
        _check(lib().klref_hierarchy_groups(self.ptr, l, None, None, _iptr(ptr), _iptr(mem)))
        return ptr, mem

    def element_matrices(self, l, kind=STIFFNESS):
        """OperatorP1::matrices / stencil: 2-d (M, 18) up + down matrices and the
        (M, 7) stencil; 3-d (M, 96) six micro-tet types of 4 x 4 and the (M, 15) stencil."""
        M = self.num_macros()
        three = getattr(self, "dim", 2) == 3
        mats = np.zeros((M, 96 if three else 18))
        st = np.zeros((M, 15 if three else 7))
        _check(lib().klref_hierarchy_element_matrices(self.ptr, l, kind, _dptr(mats), _dptr(st)))
        return mats, st

    def create_function(self, l) -> "GridFunction":
        return GridFunction(self, l)


class GridFunction(_Handle):
    """Device GridFunction (proj/include/klref/hhg.hpp:33-53): M * lattice_size(2^l) doubles."""
    _destroy = "klref_gf_destroy"

    def __init__(self, h: GridHierarchy, level: int, data: Optional[np.ndarray] = None):
        out = C.c_void_p()
        _check(lib().klref_gf_create(h.ptr, level, C.byref(out)))
        super().__init__(out.value)
        self.h = h
        self._level = level
        self.size = h.level_size(level)
        if data is not None:
            self.upload(data)

    def level(self):
        return self._level

    def upload(self, data: np.ndarray):
        a = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
        if a.size != self.size:
            raise StructuralError("grid function size mismatch")
        _check(lib().klref_gf_upload(self.ptr, _dptr(a)))

    def numpy(self) -> np.ndarray:
        out = np.empty(self.size, dtype=np.float64)
        _check(lib().klref_gf_download(self.ptr, _dptr(out)))
        return out


class Problem(_Handle):
    _destroy = "klref_problem_destroy"

    def __init__(self, kind: int, params: Optional[Sequence[float]] = None):
        out = C.c_void_p()
        _check(lib().klref_problem_create(kind, C.byref(out)))
        super().__init__(out.value)
        self.kind = kind
        if params is not None:
            p = np.ascontiguousarray(params, dtype=np.float64)
            _check(lib().klref_problem_set_params(self.ptr, _dptr(p), p.size))


@dataclass
class SolverConfig:
    """SolverConfig, proj/include/klref/multigrid.hpp:19-29 (finest_policy 0 = None,
    1 = ValidationTwoDigits on 2-d hierarchies)."""
    nu: int = 2
    pre_smooth: int = 2
    post_smooth: int = 2
    coarse_rel_tol: float = 1e-9
    coarse_abs_floor: float = 1e-12
    coarse_max_iter: int = 100000
    finest_policy: int = 0
    faithful_source: int = 0
    use_graph: int = 1
    max_extra_cycles: int = 60

    def c(self):
        return SolverConfigC(self.nu, self.pre_smooth, self.post_smooth, self.coarse_rel_tol,
                             self.coarse_abs_floor, self.coarse_max_iter, self.finest_policy,
                             self.faithful_source, self.use_graph, self.max_extra_cycles)


@dataclass
class EstimateReport:
    """EstimateReport, proj/include/klref/estimator.hpp:15-24."""
    offset: int
    base_level: int
    kind: int
    norm_coarser: float
    norm_base: float
    conv_factor: float
    eta: float
    eta_local: np.ndarray = field(default_factory=lambda: np.zeros(0))


class MultigridSolver(_Handle):
    """MultigridSolver (proj/include/klref/multigrid.hpp:62-99) on the device."""
    _destroy = "klref_solver_destroy"

    def __init__(self, h: GridHierarchy, problem: Problem, cfg: SolverConfig = SolverConfig()):
        out = C.c_void_p()
        c = cfg.c()
        _check(lib().klref_solver_create(h.ptr, problem.ptr, C.byref(c), C.byref(out)))
        super().__init__(out.value)
        self.h = h
        self.problem = problem
        self.cfg = cfg

    # -- FMG (proj/src/multigrid.cpp:248-321)
    def fmg(self) -> "FmgState":
        _check(lib().klref_solver_fmg(self.ptr))
        return FmgState(self)

    def fmg_enqueue(self):
        _check(lib().klref_solver_fmg_enqueue(self.ptr))

    def synchronize(self):
        _check(lib().klref_solver_synchronize(self.ptr))

    def stream(self) -> int:
        p = C.c_void_p()
        _check(lib().klref_solver_stream(self.ptr, C.byref(p)))
        return p.value or 0

    def launch_count(self) -> int:
        v = C.c_int()
        _check(lib().klref_solver_launch_count(self.ptr, C.byref(v)))
        return v.value

    def last_cg_iterations(self) -> int:
        v = C.c_int()
        _check(lib().klref_solver_last_cg_iterations(self.ptr, C.byref(v)))
        return v.value

    def estimate_launch_count(self) -> int:
        v = C.c_int()
        _check(lib().klref_solver_estimate_launch_count(self.ptr, C.byref(v)))
        return v.value

    def set_stream(self, stream: int):
        """Launch on a caller-owned cudaStream_t (an int handle, e.g. torch's
        ``cuda_stream``); 0 returns to the solver's own stream."""
        _check(lib().klref_solver_set_stream(self.ptr, C.c_void_p(stream or None)))

    def set_problem(self, problem: "Problem") -> int:
        """Re-tabulate the problem data on the host and copy it to the device;
        returns the host->device bytes."""
        v = C.c_int64()
        _check(lib().klref_solver_set_problem(self.ptr, problem.ptr, C.byref(v)))
        self.problem = problem
        return v.value

    def set_profiling(self, on: bool):
        _check(lib().klref_solver_set_profiling(self.ptr, int(bool(on))))

    def kernel_stats(self, kind: int = KERNEL_ALL):
        """(device ms, launches, algorithmic bytes) of one kernel kind over the
        most recent FMG + estimate (needs set_profiling(True))."""
        ms, n, b = C.c_double(), C.c_int(), C.c_double()
        _check(lib().klref_solver_kernel_stats(self.ptr, kind, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    def state_into(self, which: int, level: int, out: np.ndarray) -> np.ndarray:
        """FmgState component copied device->host into a caller buffer (e.g. pinned)."""
        if (out.size != self.h.level_size(level) or out.dtype != np.float64 or not out.flags.c_contiguous
                or not out.flags.writeable):
            raise StructuralError("state_into: buffer size / dtype mismatch")
        _check(lib().klref_solver_state_read(self.ptr, which, level, _dptr(out)))
        return out

    def state(self, which: int, level: int) -> np.ndarray:
        out = np.empty(self.h.level_size(level), dtype=np.float64)
        _check(lib().klref_solver_state_read(self.ptr, which, level, _dptr(out)))
        return out

    # -- single operations (device grid functions)
    def apply(self, kind: int, x: GridFunction, y: GridFunction):
        _check(lib().klref_apply(self.ptr, kind, x.ptr, y.ptr))

    def residual(self, u: GridFunction, b: GridFunction, r: GridFunction):
        _check(lib().klref_residual(self.ptr, u.ptr, b.ptr, r.ptr))

    def gauss_seidel(self, u: GridFunction, b: GridFunction, sweeps: int):
        _check(lib().klref_gauss_seidel(self.ptr, u.ptr, b.ptr, sweeps))

    def restrict_transpose(self, fine: GridFunction, coarse: GridFunction):
        _check(lib().klref_restrict_transpose(self.ptr, fine.ptr, coarse.ptr))

    def prolongate(self, coarse: GridFunction, fine: GridFunction):
        _check(lib().klref_prolongate(self.ptr, coarse.ptr, fine.ptr))

    def cg_level0(self, u: GridFunction, b: GridFunction):
        _check(lib().klref_cg_level0(self.ptr, u.ptr, b.ptr))

    def dot_unique(self, a: GridFunction, b: GridFunction) -> float:
        v = C.c_double()
        _check(lib().klref_dot_unique(self.ptr, a.ptr, b.ptr, C.byref(v)))
        return v.value

    def interface_sync(self, f: GridFunction, mode: int):
        _check(lib().klref_interface_sync(self.ptr, f.ptr, mode))

    # -- ExactErrorEvaluator (proj/src/fem.cpp:358-476), 2-d
    def exact_error(self):
        """ErrorNorms of ExactErrorEvaluator(h, p, L).evaluate(u_L): (global, per_macro)."""
        g = C.c_double()
        loc = np.zeros(self.h.num_macros())
        _check(lib().klref_solver_exact_error(self.ptr, C.byref(g), _dptr(loc)))
        return g.value, loc

    def exact_error_of(self, u: "GridFunction"):
        """ExactErrorEvaluator(h, p, L).evaluate(u) of a finest-level function: (global, per_macro)."""
        g = C.c_double()
        loc = np.zeros(self.h.num_macros())
        _check(lib().klref_solver_exact_error_of(self.ptr, u.ptr, C.byref(g), _dptr(loc)))
        return g.value, loc

    def solve_direct(self, level: int) -> "GridFunction":
        """MultigridSolver::solve_direct(l), proj/src/multigrid.cpp:323-357."""
        u = self.h.create_function(level)
        _check(lib().klref_solver_solve_direct(self.ptr, level, u.ptr))
        return u

    def extra_cycles(self) -> int:
        """FmgState::extra_cycles of the last fmg() (FinestPolicy::ValidationTwoDigits)."""
        v = C.c_int()
        _check(lib().klref_solver_extra_cycles(self.ptr, C.byref(v)))
        return v.value

    # -- estimator (proj/src/estimator.cpp:8-45)
    def error_estimate(self, offset: int = 1, kind: int = UNSCALED) -> EstimateReport:
        rep = EstimateReportC()
        loc = np.zeros(self.h.num_macros())
        _check(lib().klref_error_estimate(self.ptr, offset, kind, C.byref(rep), _dptr(loc)))
        return _report(rep, loc)

    def error_estimate_enqueue(self, offset: int = 1):
        _check(lib().klref_error_estimate_enqueue(self.ptr, offset))

    def error_estimate_finish(self, offset: int = 1, kind: int = UNSCALED) -> EstimateReport:
        rep = EstimateReportC()
        loc = np.zeros(self.h.num_macros())
        _check(lib().klref_error_estimate_finish(self.ptr, offset, kind, C.byref(rep), _dptr(loc)))
        return _report(rep, loc)


def shard_starts(num_macros: int, nshards: int) -> np.ndarray:
    """Contiguous macro slot ranges of the shards (starts[nshards + 1])."""
    out = np.zeros(nshards + 1, dtype=np.int32)
    _check(lib().klref_shard_starts(num_macros, nshards, _iptr(out)))
    return out


def shard_plan(h: "GridHierarchy", nshards: int, rank: int, rep_level: int, level: int):
    """Exchange plan of one shard on one level (host only): send/recv segment
    counts [nshards, colours] and the (group, slot, idx) key of every buffer
    position, for plan-consistency checks."""
    colors = C.c_int()
    _check(lib().klref_shard_plan(h.ptr, nshards, rank, rep_level, level, C.byref(colors), None, None, None, None))
    nc = colors.value
    sc = np.zeros(nshards * nc, dtype=np.int64)
    rc = np.zeros(nshards * nc, dtype=np.int64)
    _check(lib().klref_shard_plan(h.ptr, nshards, rank, rep_level, level, C.byref(colors),
                                  sc.ctypes.data_as(_PI64), rc.ctypes.data_as(_PI64), None, None))
    sk = np.full((int(sc.sum()), 3), -1, dtype=np.int32)
    rk = np.full((int(rc.sum()), 3), -1, dtype=np.int32)
    _check(lib().klref_shard_plan(h.ptr, nshards, rank, rep_level, level, C.byref(colors),
                                  sc.ctypes.data_as(_PI64), rc.ctypes.data_as(_PI64), _iptr(sk), _iptr(rk)))
    return sc.reshape(nshards, nc), rc.reshape(nshards, nc), sk, rk


class Comm(_Handle):
    """NCCL communicator of the sharded solver (one rank per GPU).  The unique
    id travels between ranks by whatever the caller uses (torch.distributed)."""
    _destroy = "klref_comm_destroy"

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().klref_comm_unique_id(buf))
        return buf.raw

    def __init__(self, nranks: int, rank: int, uid: bytes):
        if len(uid) != 128:
            raise StructuralError("NCCL unique id must be 128 bytes")
        out = C.c_void_p()
        _check(lib().klref_comm_create(nranks, rank, uid, C.byref(out)))
        super().__init__(out.value)
        self.nranks, self.rank = nranks, rank


class ShardedSolver(_Handle):
    """MultigridSolver::fmg + error_estimate over macro shards (3-d; SURVEY.md
    §8(e)).  comm=None runs `local_shards` shards in this process on one
    device (bit-identical to MultigridSolver; the parity harness); with a Comm
    this process is one shard of comm.nranks."""
    _destroy = "klref_sharded_destroy"

    def __init__(self, h: GridHierarchy, problem: Problem, cfg: SolverConfig = SolverConfig(),
                 comm: Optional[Comm] = None, local_shards: int = 1, rep_level: int = 3):
        out = C.c_void_p()
        c = cfg.c()
        _check(lib().klref_sharded_create(h.ptr, problem.ptr, C.byref(c), comm.ptr if comm else None,
                                          local_shards, rep_level, C.byref(out)))
        super().__init__(out.value)
        self.h, self.problem, self.cfg, self.comm = h, problem, cfg, comm

    def fmg(self):
        _check(lib().klref_sharded_fmg(self.ptr))

    def fmg_enqueue(self):
        _check(lib().klref_sharded_fmg_enqueue(self.ptr))

    def synchronize(self):
        _check(lib().klref_sharded_synchronize(self.ptr))

    def stream(self) -> int:
        p = C.c_void_p()
        _check(lib().klref_sharded_stream(self.ptr, C.byref(p)))
        return p.value or 0

    def counts(self):
        """(kernel launches per FMG, per estimate, bytes exchanged per FMG)."""
        a, b, x = C.c_int(), C.c_int(), C.c_double()
        _check(lib().klref_sharded_counts(self.ptr, C.byref(a), C.byref(b), C.byref(x)))
        return a.value, b.value, x.value

    def error_estimate_enqueue(self, offset: int = 1):
        _check(lib().klref_sharded_error_estimate_enqueue(self.ptr, offset))

    def error_estimate_finish(self, offset: int = 1, kind: int = UNSCALED) -> EstimateReport:
        rep = EstimateReportC()
        loc = np.zeros(self.h.num_macros())
        _check(lib().klref_sharded_error_estimate_finish(self.ptr, offset, kind, C.byref(rep), _dptr(loc)))
        return _report(rep, loc)

    def error_estimate(self, offset: int = 1, kind: int = UNSCALED) -> EstimateReport:
        self.error_estimate_enqueue(offset)
        return self.error_estimate_finish(offset, kind)

    def state(self, which: int, level: int) -> np.ndarray:
        out = np.zeros(self.h.level_size(level), dtype=np.float64)
        _check(lib().klref_sharded_state_read(self.ptr, which, level, _dptr(out)))
        return out


def _report(rep, loc):
    return EstimateReport(rep.offset, rep.base_level, rep.kind, rep.norm_coarser, rep.norm_base,
                          rep.conv_factor, rep.eta, loc)


class FmgState:
    """FmgState (proj/include/klref/multigrid.hpp:43-53); arrays stay on the device
    and are copied to the host only on access."""

    def __init__(self, solver: MultigridSolver):
        self.solver = solver
        self.L = solver.h.max_level()

    def u(self, l):
        return self.solver.state(STATE_U, l)

    def b(self, l):
        return self.solver.state(STATE_B, l)

    def w(self, l):
        """w[l] = P u[l], on level l + 1."""
        return self.solver.state(STATE_W, l + 1)


def error_estimate(state: FmgState, offset: int = 1, kind: int = UNSCALED) -> EstimateReport:
    """error_estimate(state, j, kind), proj/include/klref/estimator.hpp:26."""
    return state.solver.error_estimate(offset, kind)


# ---------------------------------------------------------------- effectivity (estimator.hpp:27-68)
@dataclass
class EquivalenceConstants:
    """EquivalenceConstants, proj/include/klref/estimator.hpp:27-31: lower * ||e|| <= eta_j <= upper * ||e||."""
    lower: float = 0.0
    upper: float = 0.0


@dataclass
class BoundsConstants:
    """BoundsConstants, proj/include/klref/estimator.hpp:40-51."""
    theta: float = 0.25
    eps: float = 0.0
    offset: int = 1
    order: int = 2
    theta_eps: float = 0.25
    equivalence: EquivalenceConstants = field(default_factory=EquivalenceConstants)
    theta_min: float = 0.25
    theta_max: float = 0.25
    spread_scaled: float = 0.0
    spread_unscaled: float = 0.0


@dataclass
class EffectivityReport:
    """EffectivityReport, proj/include/klref/estimator.hpp:56-62."""
    gamma: float = 0.0
    gamma_valid: bool = False
    gamma_local: np.ndarray = field(default_factory=lambda: np.zeros(0))
    spread: float = 0.0
    spread_valid: bool = False


def effectivity_constants(theta: float, eps: float, offset: int) -> EquivalenceConstants:
    """effectivity_constants, proj/src/estimator.cpp:47-60 (DomainError outside its range)."""
    lo, up = C.c_double(), C.c_double()
    _check(lib().klref_effectivity_constants(theta, eps, offset, C.byref(lo), C.byref(up)))
    return EquivalenceConstants(lo.value, up.value)


def local_spread_bound_scaled(theta_max: float, eps: float, offset: int) -> float:
    """local_spread_bound_scaled, proj/src/estimator.cpp:62-71."""
    v = C.c_double()
    _check(lib().klref_local_spread_bound_scaled(theta_max, eps, offset, C.byref(v)))
    return v.value


def local_spread_bound_unscaled(theta_min: float, theta_max: float, offset: int) -> float:
    """local_spread_bound_unscaled, proj/src/estimator.cpp:73-79."""
    v = C.c_double()
    _check(lib().klref_local_spread_bound_unscaled(theta_min, theta_max, offset, C.byref(v)))
    return v.value


def make_bounds(theta: float, eps: float, offset: int) -> BoundsConstants:
    """make_bounds, proj/src/estimator.cpp:81-93."""
    b = BoundsConstants(theta=theta, eps=eps, offset=offset)
    x = -math.log2(theta) if theta > 0.0 else math.inf
    # std::lround (half away from zero); a non-finite argument is left to effectivity_constants' DomainError
    b.order = int(math.copysign(math.floor(abs(x) + 0.5), x)) if math.isfinite(x) else 0
    b.theta_eps = (1.0 + eps) * theta
    b.equivalence = effectivity_constants(theta, eps, offset)
    b.theta_min = b.theta_max = theta
    b.spread_scaled = local_spread_bound_scaled(theta, eps, offset)
    b.spread_unscaled = local_spread_bound_unscaled(theta, theta, offset)
    return b


def make_bounds_from_order(order: int, eps: float, offset: int) -> BoundsConstants:
    """make_bounds_from_order, proj/src/estimator.cpp:95-99 (theta = 2^-q)."""
    b = make_bounds(2.0 ** (-float(order)), eps, offset)
    b.order = order
    return b


def effectivity_index(report: EstimateReport, exact) -> EffectivityReport:
    """effectivity_index(report, exact), proj/src/estimator.cpp:100-123; exact = (global, per_macro)
    as returned by MultigridSolver.exact_error()."""
    eg, el = exact
    loc = np.ascontiguousarray(report.eta_local, dtype=np.float64)
    ex = np.ascontiguousarray(el, dtype=np.float64)
    gl = np.zeros(loc.size)
    g, sp = C.c_double(), C.c_double()
    gv, sv = C.c_int(), C.c_int()
    _check(lib().klref_effectivity_index(report.eta, loc.size, _dptr(loc), float(eg), ex.size, _dptr(ex), C.byref(g),
                                         C.byref(gv), _dptr(gl), C.byref(sp), C.byref(sv)))
    return EffectivityReport(g.value, bool(gv.value), gl, sp.value, bool(sv.value))


def mark(rule: int, fraction: float, active_ids: Sequence[int], green_parent: Sequence[int],
         indicator: Sequence[float], reverted_ids: Sequence[int]) -> List[int]:
    """Marking of mark_and_refine (proj/src/amr.cpp:41-66): reverted-set aggregate + rule."""
    a = np.ascontiguousarray(active_ids, dtype=np.int32)
    g = np.ascontiguousarray(green_parent, dtype=np.int32)
    ind = np.ascontiguousarray(indicator, dtype=np.float64)
    rv = np.ascontiguousarray(reverted_ids, dtype=np.int32)
    out = np.zeros(max(1, rv.size), dtype=np.int32)
    cnt = C.c_int()
    _check(lib().klref_mark(rule, fraction, a.size, _iptr(a), _iptr(g), _dptr(ind), rv.size, _iptr(rv),
                            _iptr(out), C.byref(cnt)))
    return [int(v) for v in out[:cnt.value]]
