"""The reference's matrix-function KATs (proj/tests/test_poly.cpp:138-230) through the device
recurrences (apply / apply_panel on fp64 kernels): scaled identity, diagonal spectra against the
scalar power within the Taylor / Chebyshev tail bounds, 1 x 1 matrices against scalar_value,
linearity, panel vs column, size mismatch."""
import numpy as np
import pytest

from fixtures import cheb_bound, random_unit_trace_spd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dctx(R):
    return R.Context(0)


def kernel(R, a, dctx):
    return R.NormalizedKernel.from_matrix(np.asarray(a, dtype=np.float64), "fp64", ctx=dctx)


def test_int_power_scaled_identity(R, dctx):  # test_poly.cpp:138-144
    e1 = np.zeros(6)
    e1[0] = 1.0
    y = R.apply(R.MatrixFunctionSpec.int_power(2), kernel(R, np.eye(6) / 6.0, dctx), e1)
    assert np.max(np.abs(y - e1 / 36.0)) <= 1e-15


def test_taylor_diagonal(R, dctx):  # test_poly.cpp:146-159
    a = np.diag([0.5, 0.3, 0.2])
    alpha, m = 0.5, 40
    y = R.apply(R.MatrixFunctionSpec.taylor(alpha, m, 0.5), kernel(R, a, dctx), np.ones(3))
    c = R.taylor_tail_constant(alpha)
    for i, lam in enumerate((0.5, 0.3, 0.2)):
        tail = c * abs(0.2 / 0.5 - 1.0) ** (m + 1) * lam ** alpha
        assert abs(y[i] - lam ** alpha) <= tail + 1e-14


def test_chebyshev_diagonal(R, dctx):  # test_poly.cpp:161-177
    a = np.diag([0.5, 0.3, 0.2])
    alpha, u, v, m = 1.5, 0.2, 0.5, 15
    spec = R.MatrixFunctionSpec.chebyshev(alpha, m, u, v)
    vw = R.chebyshev_safeguard(u, v)
    assert vw > v  # the safeguard widened the interval
    e2 = np.array([0.0, 1.0, 0.0])
    y = R.apply(spec, kernel(R, a, dctx), e2)
    assert abs(y[1] - 0.3 ** alpha) <= cheb_bound(alpha, u, vw, m) + 1e-14
    assert abs(y[0]) <= 1e-12 and abs(y[2]) <= 1e-12


def test_one_by_one_matches_scalar_value(R, orc, dctx):  # test_poly.cpp:179-193
    rs = R.RandomStream(31)
    u, v = 0.1, 0.8
    for spec in (R.MatrixFunctionSpec.int_power(3), R.MatrixFunctionSpec.taylor(1.3, 12, v),
                 R.MatrixFunctionSpec.chebyshev(2.2, 9, u, v)):
        for _ in range(50):
            lam = u + (v - u) * rs.next_uniform()
            y = R.apply(spec, kernel(R, [[lam]], dctx), np.ones(1))
            assert y[0] == pytest.approx(R.scalar_value(spec, lam), rel=1e-13)


def test_apply_is_linear(R, orc, dctx):  # test_poly.cpp:195-210
    k = kernel(R, random_unit_trace_spd(24, 32, orc), dctx)
    g = orc.fill_gaussian(32, 24, 2)
    x, y = g[:, 0], g[:, 1]
    ca, cb = 0.7, -1.9
    for spec in (R.MatrixFunctionSpec.int_power(2), R.MatrixFunctionSpec.taylor(0.5, 15, 1.0),
                 R.MatrixFunctionSpec.chebyshev(1.5, 15, 0.0, 1.0)):
        lhs = R.apply(spec, k, ca * x + cb * y)
        rhs = ca * R.apply(spec, k, x) + cb * R.apply(spec, k, y)
        assert np.linalg.norm(lhs - rhs) <= 1e-10 * np.linalg.norm(rhs)


def test_apply_panel_agrees_with_columns(R, orc, dctx):  # test_poly.cpp:212-222
    k = kernel(R, random_unit_trace_spd(20, 33, orc), dctx)
    panel = orc.fill_gaussian(33, 20, 5)
    spec = R.MatrixFunctionSpec.chebyshev(0.8, 10, 0.0, 1.0)
    out = R.apply_panel(spec, k, panel)
    for j in range(5):
        assert np.max(np.abs(out[:, j] - R.apply(spec, k, panel[:, j]))) <= 1e-13


def test_apply_rejects_size_mismatch(R, dctx):  # test_poly.cpp:230-236
    k = kernel(R, np.eye(4) / 4.0, dctx)
    with pytest.raises(R.RenyiError) as e:
        R.apply(R.MatrixFunctionSpec.int_power(2), k, np.ones(3))
    assert e.value.kind == "size_mismatch"
