"""Device P1 assembly (npcg_fem_assemble, csrc/fem.cu) against the host
assembly that tests/test_inputs.py pins to pcgkit.fem (fem.py:42-69,
116-134): pattern and values bit for bit, signed zeros included, and the
config-1 matrix against the reference-produced golden directly."""
import numpy as np
import pytest

from golden_util import Golden
from paper_2305_16432_b200 import inputs

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def mesh_and_host(k, jitter, seed=0):
    mesh = inputs.unit_square(k, jitter, np.random.default_rng(seed))
    K, M = inputs.element_blocks(mesh)
    asm = inputs.Assembler(len(mesh.vertices), mesh.triangles)
    return mesh, K, M, asm


@pytest.mark.parametrize("k,jitter", [(8, 0.0), (24, 0.2), (33, 0.15)])
def test_pattern_and_values_bitwise(gpu, k, jitter):
    mesh, K, M, asm = mesh_and_host(k, jitter)
    dev = inputs.DeviceAssembler(len(mesh.vertices), mesh.triangles)
    np.testing.assert_array_equal(dev.row_ptr, asm.row_ptr)
    np.testing.assert_array_equal(dev.col_idx, asm.col_idx)
    Kv, Mv = asm.values(K), asm.values(M)
    np.testing.assert_array_equal(bits(dev.values(mesh.vertices, mode="K").cpu().numpy()), bits(Kv))
    np.testing.assert_array_equal(bits(dev.values(mesh.vertices, mode="M").cpu().numpy()), bits(Mv))
    s = 1e-2 * 1.0
    np.testing.assert_array_equal(bits(dev.values(mesh.vertices, mode="M+sK", scale=s).cpu().numpy()),
                                  bits(Mv + s * Kv))


def test_heat_cfg1_matches_reference_golden(gpu):
    """A = M + dt K of config 1, assembled on the device, equals the matrix
    pcgkit.fem assembled for the golden (same seeded vertices)."""
    g = Golden("cfg1_trained")
    mesh = inputs.unit_square(32, 0.2, inputs.streams(1, 1)[0])
    dev = inputs.DeviceAssembler(len(mesh.vertices), mesh.triangles)
    np.testing.assert_array_equal(dev.row_ptr, g.row_ptr)
    np.testing.assert_array_equal(dev.col_idx, g.col_idx)
    vals = dev.values(mesh.vertices, mode="M+sK", scale=1e-2 * 1.0).cpu().numpy()
    np.testing.assert_array_equal(bits(vals), bits(g.values))


def test_per_element_coefficients_batched(gpu):
    """Config-3 shape: one mesh, a distinct exp(GRF) coefficient per element and
    system, A_b = M + dt^2 K_{c_b} (inputs.wave_2d)."""
    mesh, K, M, asm = mesh_and_host(20, 0.2, seed=3)
    rng = np.random.default_rng(5)
    cent = mesh.vertices[mesh.triangles].mean(axis=1)
    B = 5
    C = np.stack([np.exp(0.5 * inputs.grf_2d(cent, rng, rng.uniform(0.05, 0.3))) for _ in range(B)], axis=1)
    dt = 1e-3
    Mv = asm.values(M)
    want = np.stack([Mv + (dt * dt) * asm.values(K * C[:, b, None, None]) for b in range(B)], axis=1)
    dev = inputs.DeviceAssembler(len(mesh.vertices), mesh.triangles)
    got = dev.values(mesh.vertices, coef=C, mode="M+sK", scale=dt * dt).cpu().numpy()
    assert got.shape == want.shape
    np.testing.assert_array_equal(bits(got), bits(want))
    # a shared coefficient vector broadcasts like the host K * c
    got1 = dev.values(mesh.vertices, coef=C[:, 2], mode="K").cpu().numpy()
    np.testing.assert_array_equal(bits(got1), bits(asm.values(K * C[:, 2, None, None])))


def test_batched_vertices(gpu):
    """Distinct jittered meshes of one topology (inputs.heat_2d with batch > 1)."""
    rngs = inputs.streams(1, 3)
    meshes = [inputs.unit_square(16, 0.2, r) for r in rngs]
    asm = inputs.Assembler(len(meshes[0].vertices), meshes[0].triangles)
    want = []
    for m in meshes:
        K, M = inputs.element_blocks(m)
        want.append(asm.values(M) + (1e-2 * 1.0) * asm.values(K))
    V = np.stack([m.vertices for m in meshes], axis=2)
    dev = inputs.DeviceAssembler(len(meshes[0].vertices), meshes[0].triangles)
    got = dev.values(V, mode="M+sK", scale=1e-2).cpu().numpy()
    np.testing.assert_array_equal(bits(got), bits(np.stack(want, axis=1)))


def test_many_contributions_use_numpy_pairwise_order(gpu):
    """A fan of 24 triangles around one vertex: its diagonal entry sums 24
    contributions, past numpy's 8-term sequential cut-over."""
    m = 24
    ang = np.linspace(0.0, 2 * np.pi, m, endpoint=False) + 0.05 * np.random.default_rng(2).standard_normal(m)
    rad = 1.0 + 0.3 * np.random.default_rng(4).random(m)
    verts = np.vstack([[0.0, 0.0], np.column_stack([rad * np.cos(ang), rad * np.sin(ang)])])
    tris = np.array([[0, 1 + i, 1 + (i + 1) % m] for i in range(m)], dtype=np.int64)
    mesh = inputs.Mesh2D(verts, tris, np.zeros(len(verts), dtype=bool))
    K, M = inputs.element_blocks(mesh)
    asm = inputs.Assembler(len(verts), tris)
    dev = inputs.DeviceAssembler(len(verts), tris)
    np.testing.assert_array_equal(bits(dev.values(verts, mode="K").cpu().numpy()), bits(asm.values(K)))
    np.testing.assert_array_equal(bits(dev.values(verts, mode="M").cpu().numpy()), bits(asm.values(M)))


def test_degenerate_and_bad_input(gpu):
    mesh, K, M, asm = mesh_and_host(4, 0.0)
    dev = inputs.DeviceAssembler(len(mesh.vertices), mesh.triangles)
    flipped = mesh.vertices.copy()
    flipped[:, 0] *= -1.0  # every triangle clockwise
    with pytest.raises(ValueError):
        dev.values(flipped)
    with pytest.raises(ValueError):
        dev.values(mesh.vertices[:-1])
    from paper_2305_16432_b200.errors import DataFormatError
    with pytest.raises(DataFormatError):
        inputs.DeviceAssembler(3, np.array([[0, 1, 5]]))


# ---- tetrahedra (configs 4 / 5) and the device Dirichlet restriction -------

def cube_and_host(k, jitter, seed=0):
    mesh = inputs.unit_cube(k, jitter, np.random.default_rng(seed))
    K, M = inputs.tet_blocks(mesh)
    asm = inputs.Assembler(len(mesh.vertices), mesh.tets)
    return mesh, K, M, asm


@pytest.mark.parametrize("k,jitter", [(3, 0.0), (6, 0.15), (9, 0.1)])
def test_tet_pattern_and_values_bitwise(gpu, k, jitter):
    """Kuhn-cube P1 tetrahedra: pattern and K / M / M + s K values bit for
    bit against inputs.tet_blocks + Assembler (runs of up to 24 contributions
    per entry: numpy's pairwise reduceat order)."""
    mesh, K, M, asm = cube_and_host(k, jitter)
    dev = inputs.DeviceAssembler(len(mesh.vertices), mesh.tets)
    np.testing.assert_array_equal(dev.row_ptr, asm.row_ptr)
    np.testing.assert_array_equal(dev.col_idx, asm.col_idx)
    Kv, Mv = asm.values(K), asm.values(M)
    np.testing.assert_array_equal(bits(dev.values(mesh.vertices, mode="K").cpu().numpy()), bits(Kv))
    np.testing.assert_array_equal(bits(dev.values(mesh.vertices, mode="M").cpu().numpy()), bits(Mv))
    s = 1e-3
    np.testing.assert_array_equal(bits(dev.values(mesh.vertices, mode="M+sK", scale=s).cpu().numpy()),
                                  bits(Mv + s * Kv))


def test_tet_per_element_coefficients_batched(gpu):
    """Config-5 shape: one mesh, kappa = exp(sigma GRF) per element and system,
    A_b = M + dt K_{kappa_b} (inputs.heat_3d)."""
    mesh, K, M, asm = cube_and_host(7, 0.15, seed=2)
    rng = np.random.default_rng(9)
    cent = mesh.vertices[mesh.tets].mean(axis=1)
    B = 3
    C = np.stack([np.exp(1.0 * inputs.grf_2d(cent, rng, rng.uniform(0.05, 0.3))) for _ in range(B)], axis=1)
    dt = 1e-3
    Mv = asm.values(M)
    dev = inputs.DeviceAssembler(len(mesh.vertices), mesh.tets)
    vals = dev.values(mesh.vertices, coef=C, mode="M+sK", scale=dt).cpu().numpy()
    for b in range(B):
        want = Mv + dt * asm.values(K * C[:, b][:, None, None])
        np.testing.assert_array_equal(bits(vals[:, b]), bits(want))
    # per-system vertices take the general kernel
    Vb = np.stack([mesh.vertices] * B, axis=2)
    vals2 = dev.values(Vb, coef=C, mode="M+sK", scale=dt).cpu().numpy()
    np.testing.assert_array_equal(bits(vals2), bits(vals))


def test_tet_inverted_element_flagged(gpu):
    mesh, _, _, _ = cube_and_host(3, 0.0)
    tets = mesh.tets.copy()
    tets[5, [1, 2]] = tets[5, [2, 1]]  # negative orientation
    dev = inputs.DeviceAssembler(len(mesh.vertices), tets)
    with pytest.raises(ValueError):
        dev.values(mesh.vertices, mode="K")


def test_poisson_3d_matrix_assembled_and_restricted_on_device(gpu):
    """Config 4 at k = 8: device tet assembly + device Dirichlet restriction
    give the matrix inputs.poisson_3d builds on the host, bit for bit, and
    the batched gather keeps the column-minor layout."""
    import torch
    prob = inputs.poisson_3d(k=8, batch=2)
    mesh = inputs.unit_cube(8, 0.15, inputs.streams(4, 1)[0])
    dev = inputs.DeviceAssembler(len(mesh.vertices), mesh.tets)
    full = dev.values(mesh.vertices, mode="K")
    from paper_2305_16432_b200.sparse import SparseMatrixCsr
    full_pat = SparseMatrixCsr(dev.n, dev.row_ptr, dev.col_idx, np.ones(dev.nnz))
    red = inputs.DeviceRestriction(full_pat, np.flatnonzero(~mesh.boundary))
    np.testing.assert_array_equal(red.row_ptr, prob.A.row_ptr)
    np.testing.assert_array_equal(red.col_idx, prob.A.col_idx)
    np.testing.assert_array_equal(bits(red.values(full).cpu().numpy()), bits(prob.A.values))
    two = torch.stack([full, 2.0 * full], dim=1)
    got = red.values(two).cpu().numpy()
    np.testing.assert_array_equal(bits(got[:, 0]), bits(prob.A.values))
    np.testing.assert_array_equal(bits(got[:, 1]), bits(2.0 * prob.A.values))
