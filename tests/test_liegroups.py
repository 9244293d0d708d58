"""Host Lie-group helpers of the public API (liegroups.py of the reference):
array functions pinned to the reference goldens, exp/log and matrix round
trips, SE(2) tangents, interpolation and retraction."""

import numpy as np

from paper_2505_03728_b200 import liegroups as lg


def test_se3_log_and_jr_inv_vs_reference(golden):
    np.testing.assert_allclose(lg.se3_log_arrays(golden["lie_q"], golden["lie_t"]), golden["lie_log"],
                               rtol=0, atol=1e-12)
    # the reference evaluates closed forms down to 1e-7 rad (cancellation ~1e-9 near 1e-4 rad);
    # the host helper switches to series below 1e-2 rad
    np.testing.assert_allclose(lg.se3_right_jacobian_inv(golden["lie_xi"]), golden["lie_jrinv"], rtol=0, atol=1e-8)


def test_exp_log_round_trips():
    rng = np.random.default_rng(0)
    xi = rng.normal(size=(50, 6))
    xi[:, 3:] *= np.geomspace(1e-9, 3.0, 50)[:, None] / np.linalg.norm(xi[:, 3:], axis=1, keepdims=True)
    q, t = lg.se3_exp_arrays(xi)
    np.testing.assert_allclose(lg.se3_log_arrays(q, t), xi, rtol=0, atol=1e-12)
    m = lg.quat_to_matrix(q)
    np.testing.assert_allclose(lg.quat_from_matrix(m), lg.quat_normalize_canonical(q), rtol=0, atol=1e-12)
    r = lg.Rotation3.from_matrix(m[7])
    np.testing.assert_allclose(r.matrix(), m[7], atol=1e-12)
    jl = lg.so3_left_jacobian(xi[:, 3:])
    np.testing.assert_allclose(jl @ lg.so3_left_jacobian_inv(xi[:, 3:]), np.broadcast_to(np.eye(3), jl.shape),
                               atol=1e-12)
    np.testing.assert_allclose(lg.skew([1.0, 2.0, 3.0]) @ [4.0, 5.0, 6.0], np.cross([1, 2, 3], [4, 5, 6]))


def test_se3_adjoint_transports_twists():
    rng = np.random.default_rng(1)
    a = lg.Transform3.exp(rng.normal(size=6))
    xi = rng.normal(size=6) * 0.3
    lhs = a.compose(lg.Transform3.exp(xi)).compose(a.inverse()).log()
    rhs = lg.se3_adjoint(a.rotation.wxyz, a.translation) @ xi
    np.testing.assert_allclose(lhs, rhs, atol=1e-12)


def test_se2_and_helpers():
    for d in ([0.3, -0.2, 0.7], [1.0, 2.0, 1e-9], [0.0, 0.0, -2.5]):
        t = lg.Transform2.exp(d)
        np.testing.assert_allclose(t.log(), d, atol=1e-12)
    a = lg.Transform3.exp([0.1, 0.2, 0.3, 0.4, -0.2, 0.1])
    b = lg.Transform3.exp([-0.3, 0.1, 0.5, -0.1, 0.6, 0.2])
    np.testing.assert_allclose(lg.interpolate(a, b, 0.0).matrix(), a.matrix(), atol=1e-12)
    np.testing.assert_allclose(lg.interpolate(a, b, 1.0).matrix(), b.matrix(), atol=1e-12)
    assert lg.tangent_dim(a) == 6 and lg.tangent_dim(lg.Transform2.identity()) == 3 and lg.tangent_dim(np.zeros(7)) == 7
    np.testing.assert_allclose(lg.local_update(a, np.zeros(6)).matrix(), a.matrix(), atol=1e-15)
    np.testing.assert_allclose(lg.local_update(np.ones(3), np.ones(3)), 2 * np.ones(3))
    np.testing.assert_allclose(lg.apply(a, [1.0, 0.0, 0.0]), a.apply([1.0, 0.0, 0.0]))
