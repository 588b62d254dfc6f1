"""Pin the oracle (oracle/port.py + oracle/kernels.c) against golden vectors
produced by the reference itself (tests/golden/make_golden.py). CPU only.

Bitwise where the oracle restates the same numpy / sequential-loop
arithmetic on the same host; the PCG history comparison is bitwise too,
since the port performs the same operations in the same order."""
import numpy as np
import pytest

from golden_util import NAMES, Golden, params_sha
from oracle import port


@pytest.fixture(scope="module", params=NAMES)
def golden(request):
    return Golden(request.param)


def _A(g, values=None):
    return port.Csr(g.n, g.row_ptr, g.col_idx, g.values if values is None else values)


def test_params_recipe_matches_reference(golden):
    hp, params = golden.params()
    if golden.meta["weights"] == "trained":
        return
    assert params_sha(params) == golden.meta["params_sha256"]
    stored = golden.stored_params()
    for k, v in stored.items():
        np.testing.assert_array_equal(params[k], v)


def test_spmv_and_apply_inverse_probe_bitwise(golden):
    if golden.name.startswith("cfg1"):
        c = golden.case(0)
        A = _A(golden)
        np.testing.assert_array_equal(port.spmv(A, c["probe_r"]), c["probe_Ar"])
        hp, params = golden.params()
        F = port.build_learned(hp, params, A, golden.rhs[:, 0])
        np.testing.assert_array_equal(F.apply_inverse(c["probe_r"]), c["probe_z"])


def test_gnn_factor_bitwise(golden):
    hp, params = golden.params()
    if golden.name.startswith("cfg3"):
        vb = golden.z["values_batch"]
        for s in range(vb.shape[1]):
            c = golden.case(s)
            A = _A(golden, np.ascontiguousarray(vb[:, s]))
            g = port.graph_from_system(A, golden.rhs[:, s])
            M, _ = port.gnn_run(hp, params, g)
            np.testing.assert_array_equal(M, c["M"])
            np.testing.assert_array_equal(port.symmetrize(M, g), c["lower"])
        return
    A = _A(golden)
    g = port.graph_from_system(A, golden.rhs[:, 0])
    M, x0 = port.gnn_run(hp, params, g)
    ref_M = golden.case(0)["M"] if "c0_M" in golden.z else golden.z["M"]
    ref_L = golden.case(0)["lower"] if "c0_lower" in golden.z else golden.z["lower"]
    np.testing.assert_array_equal(M, ref_M)
    np.testing.assert_array_equal(port.symmetrize(M, g), ref_L)
    if x0 is not None and "c0_x0" in golden.z and golden.z["c0_x0"].size:
        np.testing.assert_array_equal(x0, golden.z["c0_x0"])


def test_pcg_bitwise(golden):
    hp, params = golden.params()
    thr = tuple(golden.meta["thresholds"])
    max_iter = golden.meta.get("max_iter")
    for s in range(golden.n_cases):
        c = golden.case(s)
        if golden.name.startswith("cfg3"):
            A = _A(golden, np.ascontiguousarray(golden.z["values_batch"][:, s]))
            F = port.assemble(c["lower"], A)
        else:
            A = _A(golden)
            lower = c["lower"] if "lower" in c else golden.z["lower"]
            F = port.assemble(lower, A)
        x, rep = port.pcg_solve(A, golden.rhs[:, s], F, thresholds=thr, max_iter=max_iter)
        assert rep.iterations == int(c["iterations"])
        assert rep.converged == bool(c["converged"])
        np.testing.assert_array_equal(x, c["x"])
        np.testing.assert_array_equal(np.array(rep.history), c["history"])
        got_to = [rep.iterations_to.get(t, -1) for t in thr]
        np.testing.assert_array_equal(got_to, c["iterations_to"])
