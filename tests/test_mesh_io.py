"""Mesh / marks output of the Python mirror against files the reference itself wrote
(proj/src/mesh_io.cpp:104-163; tests/golden/*.mesh come from the reference's write_mesh
through oracle/_ref/ref_driver)."""
import glob
import os

import numpy as np
import pytest

from paper_2508_06049_b200 import klref as K

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MESHES = sorted(glob.glob(os.path.join(GOLD, "*.mesh")))


@pytest.mark.parametrize("path", MESHES, ids=[os.path.basename(p) for p in MESHES])
def test_write_mesh_reproduces_reference_file(path, tmp_path):
    mesh = K.MacroMesh.read(path)
    out = tmp_path / "out.mesh"
    mesh.write(str(out))
    ref = [ln for ln in open(path).read().splitlines() if not ln.startswith("#")]
    got = [ln for ln in open(out).read().splitlines() if not ln.startswith("#")]
    assert got == ref  # ids, %.17g coordinates, boundary flags, element rows
    assert open(out).readline().startswith("# written ")
    again = K.MacroMesh.read(str(out))
    assert np.array_equal(again.coords, mesh.coords) and np.array_equal(again.elements, mesh.elements)


def test_marks_round_trip(tmp_path):
    p = tmp_path / "marks.txt"
    K.write_marks(str(p), [5, 2, 2, 1])
    assert K.read_marks(str(p), 6).tolist() == [1, 2, 5]
    with pytest.raises(K.IoError):
        K.read_marks(str(p), 5)  # id 5 out of range
    with pytest.raises(K.IoError):
        K.read_marks(str(tmp_path / "absent.txt"), 5)
