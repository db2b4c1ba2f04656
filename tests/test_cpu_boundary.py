"""CPU tests: the C-ABI library loads and exports every declared symbol, the
host-side hierarchy logic (groups, ownership, element matrices) and the host
marking reproduce the reference, and compute entry points fail loudly
without a device.  No kernel is launched here.
"""
import os
import re

import numpy as np
import pytest

from _golden import golden, path
from paper_2508_06049_b200 import klref as K

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "klref_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(klref_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = K.lib()
    syms = declared_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/klref_b200.h but not exported"
    # and the ctypes mirror binds exactly the declared set
    assert set(K.SIGNATURES) == set(syms)
    assert L.klref_abi_version() == 1


def test_sin_problem_matches_reference_marks_from_reference_indicator():
    """Host marking (reverted-set aggregation + rule) reproduces the reference marks
    for every step of the config-2 AMR sequence and for config 1."""
    g = golden()
    for rec in g["cfg2"]:
        marks = K.mark(K.MARK_HALF_MAX, 0.0, rec["active_ids"], rec["active_green_parent"],
                       rec["eta_local_u1"], rec["reverted_ids"])
        assert marks == rec["marks_halfmax_eta"]
        top = K.mark(K.MARK_TOP_FRACTION, 0.10, rec["active_ids"], rec["active_green_parent"],
                     rec["eta_local_u1"], rec["reverted_ids"])
        assert top == rec["marks_top10_eta"]
    c1 = g["cfg1"]
    assert K.mark(K.MARK_TOP_FRACTION, 0.10, c1["active_ids"], c1["active_green_parent"],
                  c1["exact_local"], c1["reverted_ids"]) == c1["marks_top10_exact"]
    with pytest.raises(K.StructuralError):
        K.mark(K.MARK_TOP_FRACTION, 1.5, [0], [-1], [1.0], [0])


def _node_xy(mesh, slot, n, i, j):
    c = mesh.coords[mesh.elements[slot]]
    # orient positively like MacroMesh::create
    a = 0.5 * ((c[1, 0] - c[0, 0]) * (c[2, 1] - c[0, 1]) - (c[1, 1] - c[0, 1]) * (c[2, 0] - c[0, 0]))
    if a < 0:
        c = c[[0, 2, 1]]
    return c[0] + (i / n) * (c[1] - c[0]) + (j / n) * (c[2] - c[0])


@pytest.mark.parametrize("mesh_file", ["cfg1.mesh", "cfg2_k3.mesh", "cfg2_k5.mesh"])
def test_groups_share_coordinates_and_dof_count(mesh_file):
    """Every shared-node group's members sit at the same physical point (the D2
    fix: edge groups counted from the lower-id corner), slots ascend, and the
    DoF count matches the reference formula."""
    mm = K.MacroMesh.read(path(mesh_file))
    h = K.GridHierarchy.build(mm, 4, device=False)
    M = h.num_macros()
    assert M == len(mm.elements)
    for l in range(5):
        n = 1 << l
        ptr, mem = h.groups(l)
        for g in range(len(ptr) - 1):
            ms = mem[ptr[g]:ptr[g + 1]]
            assert np.all(np.diff(ms[:, 0]) > 0)
            pts = np.array([_node_xy(mm, s, n, i, j) for s, _, i, j in ms])
            assert np.max(np.abs(pts - pts[0])) < 1e-12
            for s, idx, i, j in ms:
                assert idx == K.lattice_index(n, i, j)
        nv = len(np.unique(mm.elements))
        edges = {tuple(sorted((e[a], e[b]))) for e in mm.elements for a, b in ((0, 1), (0, 2), (1, 2))}
        dofs = nv + len(edges) * (n - 1) + M * (n - 1) * (n - 2) // 2
        assert h.dof_count(l) == dofs


def test_element_matrices_known_answers():
    """SPEC.md:221 stiffness KAT on a right isoceles macro; D1 fix: the down
    cell's matrix is positive so the level-1 stencil is [4,-1,-1,-1,-1,0,0]
     instead of all zeros; mass 1^T M 1 = |T|."""
    mm = K.MacroMesh.read(path("cfg1.mesh"))
    h = K.GridHierarchy.build(mm, 3, device=False)
    mats, st = h.element_matrices(0, K.STIFFNESS)
    kat = 0.5 * np.array([[2, -1, -1], [-1, 1, 0], [-1, 0, 1]], dtype=float)
    # macro 0 = (0,0), (.5,0), (.5,.5): the right angle sits at corner 1
    perm = [1, 0, 2]
    assert np.allclose(mats[0, :9].reshape(3, 3), kat[np.ix_(perm, perm)], atol=1e-15)
    mats1, st1 = h.element_matrices(1, K.STIFFNESS)
    for s in range(h.num_macros()):
        assert np.allclose(st1[s], [4, -1, -1, -1, -1, 0, 0], atol=1e-14) or \
            np.allclose(sorted(st1[s][1:]), sorted([-1, -1, -1, -1, 0, 0]), atol=1e-14)
        assert st1[s][0] > 0
        assert np.allclose(mats1[s, 9:].reshape(3, 3).sum(), 0.0, atol=1e-14)
        assert mats1[s, 9] > 0  # down-cell diagonal positive (D1)
    mm_, _ = h.element_matrices(2, K.MASS)
    assert np.allclose(mm_[:, :9].sum(axis=1) * 16, 0.125)  # 1^T M_T 1 = |T| / n^2, |T| = 1/8


def test_structural_errors_and_no_cpu_fallback():
    mm = K.MacroMesh.read(path("cfg1.mesh"))
    bad = K.MacroMesh(mm.coords, np.array([[0, 0, 1]], dtype=np.int32))
    with pytest.raises(K.StructuralError):
        K.GridHierarchy.build(bad, 2, device=False)
    with pytest.raises(K.StructuralError):
        K.GridHierarchy.build(mm, -1, device=False)
    three = K.MacroMesh(np.zeros((4, 3)), np.array([[0, 1, 2, 3]], dtype=np.int32), dim=3)
    with pytest.raises(K.StructuralError):
        K.Mesh(three)
    if os.environ.get("CUDA_VISIBLE_DEVICES", None) == "" or not _has_device():
        with pytest.raises(K.CudaError):
            K.GridHierarchy.build(mm, 2, device=True)


def _has_device():
    try:
        import ctypes
        rt = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int()
        return rt.cuInit(0) == 0 and rt.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


def test_threaded_host_build_equals_serial():
    """The per-level host tables are built on one thread per level (common.hpp
    parallel_levels); KB_HOST_THREADS=0 builds them in order.  Both must give the
    same groups and element matrices (2-d and 3-d)."""
    import hashlib
    import subprocess
    import sys

    code = r'''
import hashlib, os, sys
sys.path.insert(0, os.environ["KB_REPO"])
import numpy as np
from paper_2508_06049_b200 import klref as K
from paper_2508_06049_b200.meshes import kuhn_cube
hsh = hashlib.sha256()
for mesh, L in ((K.MacroMesh.read(os.path.join(os.environ["KB_REPO"], "tests", "golden", "cfg2_k3.mesh")), 5), (kuhn_cube(2), 3)):
    h = K.GridHierarchy.build(mesh, L, device=False)
    for l in range(L + 1):
        ptr, mem = h.groups(l)
        hsh.update(np.ascontiguousarray(ptr).tobytes()); hsh.update(np.ascontiguousarray(mem).tobytes())
        mats, st = h.element_matrices(l, K.STIFFNESS)
        hsh.update(np.ascontiguousarray(mats).tobytes()); hsh.update(np.ascontiguousarray(st).tobytes())
        hsh.update(str(h.dof_count(l)).encode())
print(hsh.hexdigest())
'''
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = []
    for threads in ("0", None):
        env = dict(os.environ, KB_REPO=repo)
        if threads is not None:
            env["KB_HOST_THREADS"] = threads
        else:
            env.pop("KB_HOST_THREADS", None)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-500:]
        out.append(r.stdout.strip())
    assert out[0] == out[1] and len(out[0]) == 64
