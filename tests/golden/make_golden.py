"""Generate golden fixtures from the REFERENCE mesh module (run in the build
container, where /root/reference exists; the fixtures travel, the reference
does not).

    python tests/golden/make_golden.py

Pins: Grid.dual_widths / dual_volumes (mesh.py:135-156), wrap_spacing
(:130-133), fill_ghost (:280-293), pinned_mask (:311-324),
apply_dirichlet_values (:296-308), build_grid (:167-192) and the CSV repr()
round trip (:327-391) -- the conventions the oracle's Cartesian metric mode
and the product's mesh.py must reproduce.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mesh_reference.npz")


def main():
    sys.path.insert(0, REF)
    from paracycle import mesh as ref  # noqa: the reference module, imported read-only

    rng = np.random.default_rng(20240301)
    data = {}
    cases = {
        "uniform1d": ([np.linspace(0.0, 1.0, 5)], [("dirichlet", "dirichlet")]),
        "stretched1d_periodic": ([np.cumsum(rng.uniform(0.5, 1.5, 7))], [("periodic", "periodic")]),
        "mixed2d": ([np.cumsum(rng.uniform(0.5, 1.5, 6)), np.linspace(0, 2, 5)],
                    [("dirichlet", "neumann"), ("periodic", "periodic")]),
        "mixed3d": ([np.cumsum(rng.uniform(0.5, 1.5, 5)), np.cumsum(rng.uniform(0.2, 1.0, 4)),
                     np.linspace(0, 1, 6)[:-1]],
                    [("neumann", "dirichlet"), ("dirichlet", "neumann"), ("periodic", "periodic")]),
    }
    for name, (coords, kinds) in cases.items():
        grid = ref.Grid(tuple(coords))
        faces = tuple((ref.FaceBC(lo, 0.5 if lo == "dirichlet" else 0.0), ref.FaceBC(hi, -0.25 if hi == "dirichlet" else 0.0))
                      for lo, hi in kinds)
        bc = ref.BoundaryCondition(faces)
        vals = rng.normal(size=grid.shape + (2,))
        f = ref.Field(grid, vals)
        data[f"{name}/ncoords"] = np.array([len(coords)])
        for d, c in enumerate(coords):
            data[f"{name}/coords{d}"] = np.asarray(c, float)
            data[f"{name}/dual_widths{d}"] = grid.dual_widths(d, bc)
            data[f"{name}/wrap_spacing{d}"] = np.array([grid.wrap_spacing(d)])
        data[f"{name}/kinds"] = np.array([k for pair in kinds for k in pair])
        data[f"{name}/values"] = vals
        data[f"{name}/dual_volumes"] = grid.dual_volumes(bc)
        data[f"{name}/fill_ghost"] = ref.fill_ghost(f, bc)
        data[f"{name}/pinned"] = ref.pinned_mask(grid, bc)
        data[f"{name}/dirichlet_applied"] = ref.apply_dirichlet_values(f, bc).values
    # SPEC.md:49-51 / :58-60 examples through the reference itself
    g = ref.build_grid([5], extents=[(0.0, 1.0)])
    data["kat/build_grid_5"] = g.coords[0]
    g = ref.build_grid([3], coords=[np.array([0.0, 1.0, 10.0])])
    data["kat/spacings_0_1_10"] = g.spacings[0]
    for kind in ("neumann", "periodic", "dirichlet"):
        gg = ref.Grid((np.array([0.0, 1.0, 2.0]),))
        fb = ref.BoundaryCondition(((ref.FaceBC(kind), ref.FaceBC(kind)),))
        data[f"kat/ghost_{kind}"] = ref.fill_ghost(ref.Field(gg, np.array([1.0, 2.0, 3.0])), fb)[:, 0]
    np.savez(OUT, **data)
    print("wrote", OUT, len(data), "arrays")


if __name__ == "__main__":
    main()
