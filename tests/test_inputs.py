"""Our vectorised input generators reproduce the reference's own assembly
(goldens assembled by pcgkit.fem on the same vertices) bitwise. CPU only."""
import numpy as np

from golden_util import Golden
from paper_2305_16432_b200 import inputs


def test_heat_cfg1_matches_reference_assembly():
    g = Golden("cfg1_trained")
    p = inputs.heat_2d(k=32)
    np.testing.assert_array_equal(p.A.row_ptr, g.row_ptr)
    np.testing.assert_array_equal(p.A.col_idx, g.col_idx)
    np.testing.assert_array_equal(p.A.values, g.values)
    np.testing.assert_array_equal(p.rhs[:, 0], g.rhs[:, 0])


def test_poisson_dirichlet_matches_reference_assembly():
    g = Golden("cfg2_small_f64")
    p = inputs.poisson_2d(k=64, batch=g.rhs.shape[1])
    np.testing.assert_array_equal(p.A.row_ptr, g.row_ptr)
    np.testing.assert_array_equal(p.A.col_idx, g.col_idx)
    np.testing.assert_array_equal(p.A.values, g.values)
    np.testing.assert_array_equal(p.rhs, g.rhs)


def test_wave_per_element_coefficient_matches_reference_assembly():
    g = Golden("cfg3_small_f64")
    p = inputs.wave_2d(k=48, batch=2)
    np.testing.assert_array_equal(p.A.row_ptr, g.row_ptr)
    np.testing.assert_array_equal(p.values, g.z["values_batch"])
    np.testing.assert_array_equal(p.rhs, g.rhs)


def test_assembled_matrices_are_bitwise_symmetric():
    for p in (inputs.heat_2d(k=12), inputs.poisson_2d(k=12, batch=1)):
        A = p.A
        dense = A.to_dense()
        np.testing.assert_array_equal(dense, dense.T)
        assert np.all(A.diagonal() > 0)


def test_sizes_of_the_configs():
    """Topology sizes quoted in BASELINE.json / SURVEY.md Appendix B."""
    m = inputs.unit_square(256)
    assert len(m.vertices) == 66049
    asm = inputs.Assembler(len(m.vertices), m.triangles)
    assert len(asm.col_idx) == 460289
    free = np.flatnonzero(~m.boundary)
    assert len(free) == 65025


def test_kuhn_cube_p1_tetrahedra():
    """3-D generator (configs 4, 5): bitwise symmetric SPD matrices, exact P1
    identities (K 1 = 0, x'Kx = volume, total mass = volume)."""
    mesh = inputs.unit_cube(6, 0.15, np.random.default_rng(0))
    assert mesh.tets.shape == (6 * 6 ** 3, 4)
    K, M = inputs.tet_blocks(mesh)
    asm = inputs.Assembler(len(mesh.vertices), mesh.tets)
    Kv, Mv = asm.values(K), asm.values(M)
    Km = asm.matrix(Kv)
    ones = np.ones(Km.n)
    assert np.abs(inputs._host_spmv(Km, ones)).max() < 1e-14
    x = mesh.vertices[:, 0]
    assert abs(x @ inputs._host_spmv(Km, x) - 1.0) < 1e-13
    assert abs(Mv.sum() - 1.0) < 1e-13
    for p in (inputs.poisson_3d(k=6, batch=2), inputs.heat_3d(k=5, batch=2)):
        A = p.A
        dense = A.to_dense()
        np.testing.assert_array_equal(dense, dense.T)
        assert np.linalg.eigvalsh(dense).min() > 0.0
    assert inputs.poisson_3d(k=6, batch=1).A.n == 5 ** 3
    assert inputs.heat_3d(k=5, batch=1).A.n == 6 ** 3
