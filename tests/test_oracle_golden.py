"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference.

The fixtures in tests/golden/ were written by tests/golden/make_golden.py, which
imports the reference (tomokit) itself.  The C restatement of the numba kernels
is expected to be BIT-identical (same float64 operation order, no FMA); the
numpy host logic (geometry, filters) to within float64 round-off.
"""

import numpy as np
import pytest

pytestmark = []


def _bits(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape
    return a.tobytes() == b.tobytes()


class TestGeometry:
    def test_circular_matrices(self, golden, oracle):
        g = golden("geometry")
        m = oracle.circular_matrices(8, 2 * np.pi, 1200.0, 750.0, (12, 12), (1.6, 1.6))
        np.testing.assert_allclose(m, g["mats"], rtol=0, atol=1e-9)
        m4 = oracle.circular_matrices(720, 2 * np.pi, 1200.0, 750.0, (1024, 1024), (0.6, 0.6))
        np.testing.assert_allclose(m4, g["mats4"], rtol=0, atol=1e-7)

    def test_sources_and_inverse(self, golden, oracle):
        g = golden("geometry")
        s, mi = oracle.cone_rays(g["mats"])
        assert _bits(s, g["sources"])
        assert _bits(mi, g["minv"])

    def test_from_raw(self, golden, oracle):
        g = golden("geometry")
        np.testing.assert_allclose(oracle.normalize_raw(g["raw"]), g["from_raw"], atol=1e-12)

    def test_angles(self, golden, oracle):
        assert _bits(oracle.circular_angles(24, 2 * np.pi), golden("geometry")["angles"])


class TestKernelsBitExact:
    def test_parallel(self, golden, oracle):
        g = golden("parallel2d")
        assert _bits(oracle.forward_parallel_2d(g["x"], (1.0, 1.0), g["angles"], 48, 1.0, 0.5), g["fp"])
        assert _bits(oracle.forward_parallel_2d(g["sl"], (1.0, 1.0), g["angles"], 48, 1.0, 0.5), g["fp_sl"])
        assert _bits(oracle.forward_parallel_2d(g["x"], (1.0, 1.0), g["angles"], 48, 1.0, 1.0), g["fp_step1"])
        assert _bits(oracle.back_parallel_2d(g["y"], g["angles"], 1.0, (32, 32), (1.0, 1.0)), g["bp"])
        st = oracle.step_of((0.7, 1.3))
        assert _bits(oracle.forward_parallel_2d(g["x2"], (0.7, 1.3), g["angles2"], 37, 0.9, st), g["fp2"])
        assert _bits(oracle.back_parallel_2d(g["y2"], g["angles2"], 0.9, (20, 28), (0.7, 1.3)), g["bp2"])

    def test_fan(self, golden, oracle):
        g = golden("fan2d")
        a = g["angles"]
        assert _bits(oracle.forward_fan_2d(g["x"], (1.0, 1.0), a, 1200.0, 750.0, 64, 1.6, 0.5), g["fp"])
        assert _bits(oracle.back_fan_2d(g["y"], a, 1200.0, 750.0, 1.6, (32, 32), (1.0, 1.0)), g["bp"])
        assert _bits(oracle.back_fan_2d(g["y"], a, 1200.0, 750.0, 1.6, (32, 32), (1.0, 1.0), True), g["bpw"])

    def test_cone(self, golden, oracle):
        g = golden("cone3d")
        sp = (1.0, 1.0, 1.0)
        assert _bits(oracle.forward_cone_3d(g["x"], sp, g["mats"], (12, 12), 0.5), g["fp"])
        assert _bits(oracle.forward_cone_3d(g["sl"], sp, g["mats"], (12, 12), 0.5), g["fp_sl"])
        assert _bits(oracle.back_cone_3d(g["y"], g["mats"], 750.0, (16, 16, 16), sp), g["bp"])
        assert _bits(oracle.back_cone_3d(g["y"], g["mats"], 750.0, (16, 16, 16), sp, True), g["bpw"])

    def test_cone_general_trajectories(self, golden, oracle):
        g = golden("cone3d_general")
        sp = (1.1, 0.9, 1.0)
        step = oracle.step_of(sp)
        assert _bits(oracle.forward_cone_3d(g["xh"], sp, g["mats_helix"], (10, 14), step), g["fp_h"])
        assert _bits(oracle.back_cone_3d(g["yh"], g["mats_helix"], 750.0, (14, 18, 16), sp, True), g["bp_h"])
        sp = (1.0, 1.0, 1.0)
        assert _bits(oracle.forward_cone_3d(g["xt"], sp, g["mats_tilt"], (12, 12), 0.5), g["fp_t"])
        assert _bits(oracle.back_cone_3d(g["yt"], g["mats_tilt"], 750.0, (12, 12, 12), sp, True), g["bp_t"])

    def test_thread_count_does_not_change_bits(self, golden, oracle):
        # reference test_projectors.py:377-387, restated for the C oracle
        g = golden("cone3d")
        n0 = oracle.num_threads()
        outs = []
        for n in sorted({1, max(2, n0)}):
            oracle.set_num_threads(n)
            outs.append(oracle.forward_cone_3d(g["x"], (1.0, 1.0, 1.0), g["mats"], (12, 12), 0.5).tobytes())
        oracle.set_num_threads(n0)
        assert all(o == outs[0] for o in outs)


class TestFilters:
    @pytest.mark.parametrize("kind", ["ramp", "shepp_logan", "cosine"])
    @pytest.mark.parametrize("width,sp", [(12, 1.0), (48, 0.625), (100, 1.3), (1024, 0.375)])
    def test_weights(self, golden, oracle, kind, width, sp):
        np.testing.assert_allclose(oracle.filter_weights(kind, width, sp), golden("filters")[f"{kind}_{width}"],
                                   rtol=1e-13, atol=1e-13 * sp ** -2)

    def test_fft_filter(self, golden, oracle):
        g = golden("filters")
        w = oracle.filter_weights("shepp_logan", 48, 0.625)
        np.testing.assert_allclose(oracle.fft_filter(g["rows"], w, 0.625), g["rows_filtered"], atol=1e-12)

    def test_pipelines(self, golden, oracle):
        g = golden("cone3d")
        sp = (1.0, 1.0, 1.0)
        f = oracle.filter_stage_cone(g["y"], 1200.0, 750.0, (1.6, 1.6), "shepp_logan")
        np.testing.assert_allclose(f, g["filt"], rtol=0, atol=1e-6 * np.abs(g["filt"]).max())
        fdk = oracle.fdk_cone_3d(g["y"], g["mats"], 1200.0, 750.0, (1.6, 1.6), (16, 16, 16), sp, "shepp_logan")
        np.testing.assert_allclose(fdk, g["fdk"], rtol=0, atol=1e-6 * np.abs(g["fdk"]).max())
        p = golden("parallel2d")
        fb = oracle.fbp_parallel_2d(p["y"], p["angles"], 1.0, (32, 32), (1.0, 1.0), "shepp_logan")
        np.testing.assert_allclose(fb, p["fbp"], rtol=0, atol=1e-6 * np.abs(p["fbp"]).max())
        f2 = golden("fan2d")
        ff = oracle.fbp_fan_2d(f2["y"], f2["angles"], 1200.0, 750.0, 1.6, (32, 32), (1.0, 1.0), "cosine")
        np.testing.assert_allclose(ff, f2["fbp"], rtol=0, atol=1e-6 * np.abs(f2["fbp"]).max())


class TestTransposeOracles:
    def test_parallel_transpose_is_dense_transpose(self, golden, oracle):
        g = golden("dense")
        A = g["A_par"]
        rng = np.random.default_rng(5)
        y = rng.standard_normal(A.shape[0])
        got = oracle.forward_parallel_2d_T(y.reshape(3, 9), (5, 6), (1.0, 1.0), g["ang_par"], 1.0, 0.5)
        np.testing.assert_allclose(got.ravel(), A.T @ y, atol=1e-12)

    def test_cone_transposes_are_dense_transposes(self, golden, oracle):
        g = golden("dense")
        A, B = g["A_cone"], g["B_cone"]
        rng = np.random.default_rng(6)
        y = rng.standard_normal(A.shape[0])
        got = oracle.forward_cone_3d_T(y.reshape(3, 5, 6), (4, 5, 6), (1.0, 1.0, 1.0), g["mats_cone"], 0.5)
        np.testing.assert_allclose(got.ravel(), A.T @ y, atol=1e-12)
        x = rng.standard_normal(B.shape[0])
        got = oracle.back_cone_3d_T(x.reshape(4, 5, 6), g["mats_cone"], 750.0, (5, 6), (1.0, 1.0, 1.0))
        np.testing.assert_allclose(got.ravel(), B.T @ x, atol=1e-12)
