"""Generates tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libdgref.so, built from /root/reference/proj/src by
oracle/ref/Makefile). Run in the build container (the reference sources are
not on the GPU box); the fixtures are committed.

Cases follow BASELINE.json's configs at parity-test sizes:
  * inputs: std::mt19937(seed) + uniform(-1,1) in canonical numbering
    (reference tests/test_helpers.hpp:11-19);
  * y = A x through RankOperator::apply, one rank or R threaded ranks with
    the GhostExchanger transport (tests/test_ghost_exchange.cpp:63-87);
  * faces, owners, ghost cells and exchange plans per rank (bit-exact
    indexing pins);
  * g3 geometry arrays from precompute_geometry;
  * for the BASELINE vertex deformation and the folded a(x) coefficient,
    which the reference mesh cannot express, the geometry is computed by the
    C restatement (oracle/dgoracle.c, itself pinned bit-exact against
    precompute_geometry on reference meshes) and injected into the
    reference RankOperator.

usage: python tests/golden/make_golden.py [--other-bases | --advection]
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402
from oracle import reflib as R  # noqa: E402

GEOM = ["inv_jac_t", "jxw", "face_jxw", "face_jni", "face_jne", "penalty",
        "cell_volume"]


def world_arrays(w, n_ranks, prefix="", basis="gl"):
    out = {}
    f = w.faces()
    out.update({prefix + "face_" + k: v for k, v in f.items()})
    for r in range(n_ranks):
        lay = w.layout(r)
        out[f"{prefix}r{r}_ghosts"] = lay["ghost_cells"]
        out[f"{prefix}r{r}_ghost_owner"] = lay["ghost_owner"]
        out[f"{prefix}r{r}_info"] = np.array(
            [lay["owned_cell_begin"], lay["n_owned_cells"], lay["owned_size"],
             lay["total_size"]], np.int64)
        for which in ("send", "recv"):
            pl = w.plans(r, which)
            out[f"{prefix}r{r}_{which}_neighbors"] = np.array(
                [p["neighbor"] for p in pl], np.int32)
            for i, p in enumerate(pl):
                out[f"{prefix}r{r}_{which}{i}_cells"] = p["cells"]
                if basis != "gl" or getattr(w, "kind", "laplacian") == "advection":
                    # Hermite: two layers per coupled face, nodal values: one
                    # (ghost_exchange.cpp:46-96)
                    out[f"{prefix}r{r}_{which}{i}_offsets"] = p["offsets"]
                    out[f"{prefix}r{r}_{which}{i}_dofs"] = p["dofs"]
                    continue
                # GL + first derivatives: whole cells travel
                dpc = w.dofs_per_cell
                assert np.array_equal(p["offsets"], np.arange(len(p["cells"]) + 1) * dpc)
                assert np.array_equal(p["dofs"], np.tile(np.arange(dpc), len(p["cells"])))
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


BASIS_ID = {"gl": 0, "gauss": 1, "hermite": 2}


def reference_case(name, d, cells, p, periodic, amplitude, m, n_ranks, seeds,
                   dense=False, geometry=True, basis="gl", kind="laplacian",
                   velocity=(1.0, 1.0, 1.0), velocity_field=0):
    w = R.World(d, cells, p, n_ranks=n_ranks, amplitude=amplitude,
                mapping_degree=m, periodic=periodic, basis=basis, kind=kind,
                velocity=velocity, velocity_field=velocity_field)
    arr = dict(meta=np.array([d, *cells, p, int(periodic), m, n_ranks], np.int64),
               amplitude=np.array(amplitude))
    if basis != "gl":
        arr["basis"] = np.array(BASIS_ID[basis])
    if kind == "advection":
        arr["advection"] = np.array([*velocity, velocity_field], np.float64)
    for s in seeds:
        x = R.random_vector(w.n_dofs, s)
        arr[f"x{s}"] = x
        arr[f"y{s}"] = w.apply(x)
    arr.update(world_arrays(w, n_ranks, basis=basis))
    if geometry:
        for g in GEOM:
            arr["geo_" + g] = w.geometry(g)
    arr["compressed"] = np.array(w.compressed)
    if dense:
        arr["A"] = w.assemble()
    save(name, **arr)


def injected_case(name, d, cells, p, periodic, eps, coefficient, n_ranks, seeds,
                  basis="gl"):
    P = O.Problem(d, cells, p, periodic=periodic, deform=("vertex", eps),
                  coefficient=coefficient, n_ranks=n_ranks)
    geo = {k: P.geom[k] for k in ("inv_jac_t", "jxw", "face_jxw", "face_jni",
                                  "face_jne", "penalty")}
    geo["compressed"] = False
    w = R.World(d, cells, p, n_ranks=n_ranks, periodic=periodic, geometry=geo, basis=basis)
    arr = dict(meta=np.array([d, *cells, p, int(periodic), 1, n_ranks], np.int64),
               eps=np.array(eps), coefficient=np.array(int(coefficient)))
    if basis != "gl":
        arr["basis"] = np.array(BASIS_ID[basis])
    for s in seeds:
        x = R.random_vector(w.n_dofs, s)
        arr[f"x{s}"] = x
        arr[f"y{s}"] = w.apply(x)
    arr.update(world_arrays(w, n_ranks, basis=basis))
    for g in GEOM:
        arr["geo_" + g] = P.geom[g]
    save(name, **arr)


def basics():
    arr = {}
    for n in range(1, 13):
        p, w = R.gauss(n)
        arr[f"gauss{n}_p"], arr[f"gauss{n}_w"] = p, w
        if n >= 2:
            p, w = R.gauss(n, lobatto=True)
            arr[f"lobatto{n}_p"], arr[f"lobatto{n}_w"] = p, w
    for p in range(1, 11):
        sm = R.shape_matrices(p)
        for k, v in sm.items():
            arr[f"p{p}_{k}"] = v
    for seed in (0, 1, 2, 3, 4):
        arr[f"rng{seed}"] = R.random_vector(1000, seed)
    save("basics", **arr)


def bases():
    """Shape matrices of the other two bases (basis.cpp:116-180,261-325)."""
    arr = {}
    for p in range(1, 11):
        for b in ("gauss", "hermite"):
            if b == "hermite" and p < 3:
                continue
            for k, v in R.shape_matrices(p, b).items():
                arr[f"{b}_p{p}_{k}"] = v
    save("basics_bases", **arr)


def other_bases():
    """The reference's default Laplacian basis for p >= 3 is Hermite-like
    (operators.cpp:27-41): 2-layer face reads and exchange plans."""
    bases()
    reference_case("herm3d_p3_m2", 3, [3, 3, 3], 3, False, 0.05, 2, 1, [21], basis="hermite")
    reference_case("herm3d_p5_m2_r3", 3, [3, 3, 4], 5, False, 0.05, 2, 3, [22],
                   basis="hermite")
    reference_case("herm2d_p4_m3_r2", 2, [4, 5], 4, False, 0.06, 3, 2, [23], basis="hermite")
    reference_case("herm3d_periodic_cart_p6_r2", 3, [3, 3, 3], 6, True, 0.0, 1, 2, [24],
                   basis="hermite")
    reference_case("herm2d_p10_m2", 2, [3, 3], 10, False, 0.05, 2, 1, [25], basis="hermite")
    reference_case("herm2d_p3_dense", 2, [2, 3], 3, False, 0.05, 2, 1, [26], dense=True,
                   basis="hermite")
    injected_case("herm_c4_vertex_coef_p5_r2", 3, [3, 3, 3], 5, False, 0.1, True, 2, [27],
                  basis="hermite")
    reference_case("gauss3d_p3_m2_r2", 3, [3, 2, 2], 3, False, 0.05, 2, 2, [28], basis="gauss")
    reference_case("gauss2d_p2_periodic", 2, [4, 4], 2, True, 0.0, 1, 1, [29], basis="gauss")


def advection():
    """The advection operator (OperatorKind::advection), the paper's other
    operator: constant and variable transport fields, one-layer plans."""
    c = (0.85, 0.6, 0.35)
    reference_case("adv3d_p3_m2", 3, [3, 3, 3], 3, False, 0.05, 2, 1, [31], kind="advection",
                   velocity=c)
    reference_case("adv3d_p4_m2_r3", 3, [3, 3, 4], 4, False, 0.05, 2, 3, [32],
                   kind="advection", velocity=c)
    reference_case("adv2d_periodic_p5_m3_r2", 2, [5, 4], 5, True, 0.06, 3, 2, [33],
                   kind="advection", velocity=(-0.4, 0.9, 0.0))
    reference_case("adv3d_cart_p6_r2", 3, [3, 3, 3], 6, False, 0.0, 1, 2, [34],
                   kind="advection", velocity=c)
    reference_case("adv2d_field_p3_m2_r2", 2, [4, 4], 3, False, 0.05, 2, 2, [35],
                   kind="advection", velocity_field=1)
    reference_case("adv3d_field_p2_m2", 3, [3, 2, 3], 2, False, 0.04, 2, 1, [36],
                   kind="advection", velocity_field=1)
    reference_case("adv_gauss3d_p3_m2_r2", 3, [3, 2, 2], 3, False, 0.05, 2, 2, [37],
                   kind="advection", velocity=c, basis="gauss")


def main():
    if "--advection" in sys.argv:
        advection()
        return
    if "--other-bases" in sys.argv:
        other_bases()
        return
    basics()
    # C1 shape (3D periodic Cartesian, p=3), reduced to 4^3 cells; 2 ranks
    reference_case("c1_periodic_cart_p3", 3, [4, 4, 4], 3, True, 0.0, 1, 1, [0, 11])
    reference_case("c1_periodic_cart_p3_r2", 3, [4, 4, 4], 3, True, 0.0, 1, 2, [0])
    # C2 shape (2D Dirichlet Cartesian), degree sweep p=1..10 on 8^2 cells
    for p in range(1, 11):
        reference_case(f"c2_dirichlet_cart_p{p}", 2, [8, 8], p, False, 0.0, 1, 1, [1],
                       geometry=(p in (1, 5, 10)))
    # reference-deformed meshes (curved mapping m = 2, 3), with rank splits
    reference_case("def2d_p3_m3", 2, [3, 3], 3, False, 0.07, 3, 1, [5], dense=True)
    reference_case("def2d_periodic_p2_r4", 2, [4, 4], 2, True, 0.05, 2, 4, [7])
    reference_case("def3d_p3_m2_r2", 3, [2, 2, 2], 3, False, 0.05, 2, 2, [41])
    reference_case("def3d_p2_m3_r7", 3, [4, 4, 4], 2, False, 0.06, 3, 7, [3])
    reference_case("cart3d_ragged_p4_r3", 3, [3, 2, 4], 4, True, 0.0, 1, 3, [9])
    # C3 shape (BASELINE vertex deformation, p=4) reduced to 4^3 cells
    injected_case("c3_vertex_p4", 3, [4, 4, 4], 4, False, 0.1, False, 1, [2])
    injected_case("c3_vertex_p4_r3", 3, [4, 4, 4], 4, False, 0.1, False, 3, [2])
    # C4 shape (vertex deformation + folded a(x), p=5) reduced to 3^3 cells
    injected_case("c4_vertex_coef_p5_r2", 3, [3, 3, 3], 5, False, 0.1, True, 2, [3])
    # C5 shape (Cartesian Dirichlet, p=6) reduced to 3^3 cells
    reference_case("c5_cart_p6", 3, [3, 3, 3], 6, False, 0.0, 1, 1, [4])


if __name__ == "__main__":
    main()
    if "--other-bases" not in sys.argv and "--advection" not in sys.argv:
        other_bases()
        advection()
