"""Coarse (macro) meshes of the BASELINE.json configurations (host inputs).

2-d meshes come from the patched reference itself (tests/golden/*.mesh, the
reference's mesh_io format); the 3-d configurations use the Kuhn cube
triangulation the reference's waves3d_initial_mesh builds
(proj/src/problems.cpp:111-136), generalised to N^3 cubes.
"""
import numpy as np

from .klref import MacroMesh

# the six tetrahedra of a Kuhn cube: paths (0,0,0) -> (1,1,1) along the axis permutations
_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def kuhn_cube(N: int) -> MacroMesh:
    """Unit cube split into N^3 cubes x 6 Kuhn tetrahedra; vertex id i + (N+1) j + (N+1)^2 k,
    slot order cube-major (k, j, i), tets in axis-permutation order."""
    n1 = N + 1
    g = np.arange(n1) / N
    coords = np.array([[g[i], g[j], g[k]] for k in range(n1) for j in range(n1) for i in range(n1)])

    def vid(i, j, k):
        return i + n1 * j + n1 * n1 * k

    tets = []
    for k in range(N):
        for j in range(N):
            for i in range(N):
                for p in _PERMS:
                    c = [0, 0, 0]
                    t = [vid(i, j, k)]
                    for ax in p:
                        c[ax] += 1
                        t.append(vid(i + c[0], j + c[1], k + c[2]))
                    tets.append(t)
    return MacroMesh(coords, np.array(tets, dtype=np.int32), 3)


def series_coefficients(seed: int = 20240817) -> np.ndarray:
    """C_abc ~ U(-1, 1), a, b, c = 1..4 (a fastest), BASELINE.json config 5."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, 64)
