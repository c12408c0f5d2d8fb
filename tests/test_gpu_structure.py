"""Level build on the B200 vs the compiled reference: mesh, DOF numbering,
CSR structure and values bit-exact (north star: "mesh, connectivity and CSR
structure bit-exact"), partition and region index sets equal."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # (name, domain, H, delta, m, levels)
    ("unit8_L4_m4", (0.0, 1.0, 0.0, 1.0), 1 / 8, 1 / 8, 4, 4),
    ("unit16_L3_m16", (0.0, 1.0, 0.0, 1.0), 1 / 16, 1 / 16, 16, 3),
    ("square_H025_m4", (-1.0, 1.0, -1.0, 1.0), 0.25, 0.25, 4, 3),
    ("rect_3x2_m1", (0.0, 3.0, -1.0, 1.0), 0.5, 0.5, 1, 3),
    # lattice steps that are NOT bitwise uniform (8 distinct x steps at level 3):
    # the generic k_assemble gather; the cases above take k_assemble_table
    ("offset_H01_m1", (0.1, 1.3, -0.2, 0.4), 0.1, 0.1, 1, 3),
]


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def make(mlg, oracle_ref, domain, H, delta, m, levels):
    cfg = mlg.RunConfig(domain=mlg.DomainRect(*domain), H=H, delta=delta, m=m, n_levels=levels,
                        nev=1)
    hy = mlg.Hierarchy(cfg)
    rh = oracle_ref.RefHierarchy(domain=domain, H=H, delta=delta, m=m, n_levels=levels, nev=1)
    hy.extend_to(levels)
    rh.extend_to(levels)
    return hy, rh


@pytest.mark.parametrize("name,domain,H,delta,m,levels", CASES)
def test_mesh_space_csr_bitexact(mlg, oracle_ref, name, domain, H, delta, m, levels):
    hy, rh = make(mlg, oracle_ref, domain, H, delta, m, levels)
    for k in range(levels + 1):
        g = hy.mesh(k)
        r = rh.mesh(k)
        assert np.array_equal(g.triangles, r["triangles"]), (name, k)
        assert np.array_equal(bits(g.vertices), bits(r["vertices"])), (name, k)
        assert np.array_equal(g.vertex_lattice, r["lattice"]), (name, k)
        assert np.array_equal(g.boundary_edges, r["boundary_edges"]), (name, k)
        if k:
            assert np.array_equal(g.parent, r["parent"]), (name, k)
        assert g.h_max == r["h_max"]
        gs, rs = hy.space(k), rh.space(k)
        for key in ("dof_lattice", "interior_dofs", "interior_index", "connectivity"):
            assert np.array_equal(getattr(gs, key), rs[key]), (name, k, key)
        for form in ("stiffness", "mass"):
            grp, gc, gv = hy.csr(k, form)
            rrp, rc, rv = rh.csr(k, form)
            assert np.array_equal(grp, rrp) and np.array_equal(gc, rc), (name, k, form)
            assert np.array_equal(bits(gv), bits(rv)), (name, k, form)


@pytest.mark.parametrize("name,domain,H,delta,m,levels", CASES)
def test_partition_and_regions(mlg, oracle_ref, name, domain, H, delta, m, levels):
    hy, rh = make(mlg, oracle_ref, domain, H, delta, m, levels)
    p = hy.partition()
    info, rects = rh.partition()
    assert [p["m"], p["side"], p["overlap_cells"], p["coarse_nx"], p["coarse_ny"]] == list(info)
    assert np.array_equal(p["blocks"], rects[:, 0])
    assert np.array_equal(p["overlaps"], rects[:, 1])
    assert np.array_equal(p["inners"], rects[:, 2])
    for k in range(levels + 1):
        for kind in ("domain", "block", "overlap", "inner", "strip"):
            js = [0] if kind in ("domain", "strip") else range(m)
            for j in js:
                for zt in (False, True):
                    assert np.array_equal(hy.region_dofs(k, kind, j, zt),
                                          rh.region_dofs(k, kind, j, zt)), (name, k, kind, j, zt)
                assert np.array_equal(hy.region_elements(k, kind, j),
                                      rh.region_elements(k, kind, j)), (name, k, kind, j)


def test_spmv_prolong_restrict_bitexact(mlg, oracle_ref):
    hy, rh = make(mlg, oracle_ref, (0.0, 1.0, 0.0, 1.0), 1 / 8, 1 / 8, 4, 3)
    rng = np.random.default_rng(20261019)
    for k in range(4):
        n = hy.level_info(k).ndofs
        x = rng.uniform(-1, 1, n)
        for form in ("stiffness", "mass"):
            assert np.array_equal(bits(hy.apply(k, form, x)), bits(rh.apply(k, form, x)))
    for a in range(3):
        for b in range(a, 4):
            x = rng.uniform(-1, 1, hy.level_info(a).ndofs)
            assert np.array_equal(bits(hy.prolong(x, a, b)), bits(rh.prolong(x, a, b)))
            y = rng.uniform(-1, 1, hy.level_info(b).ndofs)
            assert np.array_equal(bits(hy.restrict_transpose(y, b, a)),
                                  bits(rh.restrict_transpose(y, b, a)))


def test_assembly_table_equals_generic_gather(mlg, monkeypatch):
    """k_assemble_table (translation-invariant lattices) is bitwise the generic
    k_assemble gather (fespace.cpp:314-341 + sparse.cpp:24-61), and the offset
    domain falls back to the generic kernel."""
    def operators(domain, H, levels):
        cfg = mlg.RunConfig(domain=mlg.DomainRect(*domain), H=H, delta=H, m=1, n_levels=levels,
                            nev=1)
        with mlg.Hierarchy(cfg) as hy:
            hy.set_profiling(True)
            hy.extend_to(levels)
            kernel = hy.build_profile_kernel()
            return kernel, [hy.csr(levels, f) for f in ("stiffness", "mass")]

    for domain, H, levels in (((0.0, 1.0, 0.0, 1.0), 1 / 8, 5), ((-1.0, 1.0, -1.0, 1.0), 0.25, 4),
                              ((0.0, 3.0, -1.0, 1.0), 0.5, 4)):
        monkeypatch.delenv("MLG_ASSEMBLE_TABLE", raising=False)
        k1, ops1 = operators(domain, H, levels)
        monkeypatch.setenv("MLG_ASSEMBLE_TABLE", "0")
        k0, ops0 = operators(domain, H, levels)
        assert (k1, k0) == ("k_assemble_table", "k_assemble")
        for (rp1, c1, v1), (rp0, c0, v0) in zip(ops1, ops0):
            assert np.array_equal(rp1, rp0) and np.array_equal(c1, c0)
            assert np.array_equal(bits(v1), bits(v0))
    monkeypatch.delenv("MLG_ASSEMBLE_TABLE", raising=False)
    k, _ = operators((0.1, 1.3, -0.2, 0.4), 0.1, 3)
    assert k == "k_assemble"
