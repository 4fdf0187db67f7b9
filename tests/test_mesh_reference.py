"""Pin the mesh conventions of the product (paper_2403_01004_b200.mesh) and of
the oracle's Cartesian metric mode to the REFERENCE mesh.py, through golden
fixtures generated from it (tests/golden/make_golden.py) and, when the
reference tree is present, live."""
import os
import sys

import numpy as np
import pytest

from helpers import oracle_geometry
from paper_2403_01004_b200 import mesh

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "mesh_reference.npz"))
CASES = sorted({k.split("/")[0] for k in GOLD.files if not k.startswith("kat/")})


def _case(name):
    n = int(GOLD[f"{name}/ncoords"][0])
    coords = [GOLD[f"{name}/coords{d}"] for d in range(n)]
    kinds = list(GOLD[f"{name}/kinds"])
    pairs = [(kinds[2 * d], kinds[2 * d + 1]) for d in range(n)]
    faces = tuple((mesh.FaceBC(lo, 0.5 if lo == "dirichlet" else 0.0), mesh.FaceBC(hi, -0.25 if hi == "dirichlet" else 0.0))
                  for lo, hi in pairs)
    return mesh.Grid(tuple(coords)), mesh.BoundaryCondition(faces), pairs


@pytest.mark.parametrize("name", CASES)
def test_dual_cells_match_reference(name):
    grid, bc, pairs = _case(name)
    for d in range(grid.dims):
        assert np.array_equal(grid.dual_widths(d, bc), GOLD[f"{name}/dual_widths{d}"])
        assert grid.wrap_spacing(d) == GOLD[f"{name}/wrap_spacing{d}"][0]
    assert np.array_equal(grid.dual_volumes(bc), GOLD[f"{name}/dual_volumes"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_cartesian_volumes_match_reference(name):
    """The oracle's finite-volume and aligned control volumes == reference dual volumes."""
    grid, bc, pairs = _case(name)
    g = oracle_geometry(grid, bc)
    ref = GOLD[f"{name}/dual_volumes"].reshape(g.shape)
    assert np.allclose(g.volume(), ref, rtol=1e-15, atol=0)
    assert np.allclose(g.aligned_volume(), ref, rtol=1e-15, atol=0)


@pytest.mark.parametrize("name", CASES)
def test_ghost_pinned_dirichlet_match_reference(name):
    grid, bc, _ = _case(name)
    f = mesh.Field(grid, GOLD[f"{name}/values"])
    assert np.array_equal(mesh.fill_ghost(f, bc), GOLD[f"{name}/fill_ghost"])
    assert np.array_equal(mesh.pinned_mask(grid, bc), GOLD[f"{name}/pinned"])
    assert np.array_equal(mesh.apply_dirichlet_values(f, bc).values, GOLD[f"{name}/dirichlet_applied"])
    g = oracle_geometry(grid, bc)
    assert np.array_equal(g.pinned.reshape(GOLD[f"{name}/pinned"].shape), GOLD[f"{name}/pinned"])


def test_spec_mesh_kats():
    """SPEC.md:49-51, :58-60 (reproduced by the reference and by us)."""
    assert np.array_equal(mesh.build_grid([5], extents=[(0.0, 1.0)]).coords[0], GOLD["kat/build_grid_5"])
    assert np.array_equal(mesh.build_grid([3], coords=[np.array([0.0, 1.0, 10.0])]).spacings[0],
                          GOLD["kat/spacings_0_1_10"])
    g = mesh.build_grid([4, 4], extents=[(0, 1), (0, 1)])
    assert g.npoints == 16 and np.allclose(g.spacings[0], 1 / 3)
    gg = mesh.Grid((np.array([0.0, 1.0, 2.0]),))
    for kind, ghosts in (("neumann", (1, 3)), ("periodic", (3, 1)), ("dirichlet", (0, 0))):
        bc = mesh.BoundaryCondition(((mesh.FaceBC(kind), mesh.FaceBC(kind)),))
        out = mesh.fill_ghost(mesh.Field(gg, np.array([1.0, 2.0, 3.0])), bc)[:, 0]
        assert np.array_equal(out, GOLD[f"kat/ghost_{kind}"])
        assert (out[0], out[-1]) == ghosts


def test_invalid_grids():
    with pytest.raises(mesh.InvalidGridError):
        mesh.build_grid([2], extents=[(0, 1)])
    with pytest.raises(mesh.InvalidGridError):
        mesh.Grid((np.array([0.0, 2.0, 1.0]),))
    with pytest.raises(ValueError):
        mesh.BoundaryCondition(((mesh.FaceBC("periodic"), mesh.FaceBC("neumann")),))
    with pytest.raises(ValueError):
        mesh.FaceBC("robin")


def test_csv_round_trip_bit_exact(tmp_path):
    grid, bc, _ = _case("mixed3d")
    f = mesh.Field(grid, GOLD["mixed3d/values"])
    mesh.write_field_csv(f, str(tmp_path / "f.csv"))
    mesh.write_coords_csv(grid, str(tmp_path / "c.csv"))
    g = mesh.read_field_csv(str(tmp_path / "f.csv"), str(tmp_path / "c.csv"))
    assert np.array_equal(g.values, f.values)
    assert all(np.array_equal(a, b) for a, b in zip(g.grid.coords, grid.coords))


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present (GPU box)")
def test_live_reference_csv_interop(tmp_path):
    """Files written by the reference are read bit-exactly by us and vice versa."""
    sys.path.insert(0, REF)
    from paracycle import mesh as ref

    grid, bc, _ = _case("mixed2d")
    vals = GOLD["mixed2d/values"]
    ref.write_field_csv(ref.Field(ref.Grid(grid.coords), vals), str(tmp_path / "r.csv"))
    ref.write_coords_csv(ref.Grid(grid.coords), str(tmp_path / "rc.csv"))
    ours = mesh.read_field_csv(str(tmp_path / "r.csv"), str(tmp_path / "rc.csv"))
    assert np.array_equal(ours.values, vals)
    mesh.write_field_csv(mesh.Field(grid, vals), str(tmp_path / "o.csv"))
    mesh.write_coords_csv(grid, str(tmp_path / "oc.csv"))
    back = ref.read_field_csv(str(tmp_path / "o.csv"), str(tmp_path / "oc.csv"))
    assert np.array_equal(back.values, vals)
