"""GPU parity: the sm_100a kernels against the reference's golden vectors and the
float64 C oracle, within the north-star tolerance (relative L2 <= 1e-4).

All calls go through libtkb200.so (the C ABI); nothing here falls back to CPU.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-4  # north star: relative L2 <= 1e-4 on sinograms and volumes


def rel(got, want):
    got = np.asarray(got.detach().cpu().numpy() if isinstance(got, torch.Tensor) else got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


@pytest.fixture(scope="module")
def tk(cuda):
    import paper_2511_08427_b200 as tk

    return tk


def T(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float32)).cuda()


# ---------------------------------------------------------------------------
# golden vectors (produced by the reference itself)
# ---------------------------------------------------------------------------


class TestGolden:
    def test_parallel(self, tk, golden):
        g = golden("parallel2d")
        geom = tk.GeometryParallel2D((32, 32), (1.0, 1.0), 48, 1.0, g["angles"])
        assert rel(tk.forward_project(tk.Volume(g["x"], (1, 1)), geom).data, g["fp"]) < TOL
        assert rel(tk.forward_project(tk.Volume(g["sl"], (1, 1)), geom).data, g["fp_sl"]) < TOL
        assert rel(tk.forward_project(tk.Volume(g["x"], (1, 1)), geom, tk.SamplingConfig(1.0)).data,
                   g["fp_step1"]) < TOL
        assert rel(tk.back_project(tk.Sinogram(g["y"], (1.0,)), geom).data, g["bp"]) < TOL
        g2 = tk.GeometryParallel2D((20, 28), (0.7, 1.3), 37, 0.9, g["angles2"])
        assert rel(tk.forward_project(tk.Volume(g["x2"], (0.7, 1.3)), g2).data, g["fp2"]) < TOL
        assert rel(tk.back_project(tk.Sinogram(g["y2"], (0.9,)), g2).data, g["bp2"]) < TOL
        assert rel(tk.fbp_parallel_2d(tk.Sinogram(g["y"], (1.0,)), geom, "shepp_logan").data, g["fbp"]) < TOL
        assert rel(tk.fbp_parallel_2d(tk.Sinogram(g["y"], (1.0,)), geom, "ramp").data, g["fbp_ramp"]) < TOL

    def test_fan(self, tk, golden):
        g = golden("fan2d")
        geom = tk.GeometryFan2D((32, 32), (1.0, 1.0), 64, 1.6, g["angles"], sdd=1200.0, sid=750.0)
        assert rel(tk.forward_project(tk.Volume(g["x"], (1, 1)), geom).data, g["fp"]) < TOL
        y = tk.Sinogram(g["y"], (1.6,))
        assert rel(tk.back_project(y, geom).data, g["bp"]) < TOL
        assert rel(tk.back_project(y, geom, fdk_weighting=True).data, g["bpw"]) < TOL
        assert rel(tk.fbp_fan_2d(y, geom, "cosine").data, g["fbp"]) < TOL

    def test_cone(self, tk, golden):
        g = golden("cone3d")
        geom = tk.circular_cone_geometry((16, 16, 16), (1, 1, 1), (12, 12), (1.6, 1.6), 8, 2 * np.pi,
                                         1200.0, 750.0)
        assert rel(tk.forward_project(tk.Volume(g["x"], (1, 1, 1)), geom).data, g["fp"]) < TOL
        assert rel(tk.forward_project(tk.Volume(g["sl"], (1, 1, 1)), geom).data, g["fp_sl"]) < TOL
        y = tk.Sinogram(g["y"], (1.6, 1.6))
        assert rel(tk.back_project(y, geom).data, g["bp"]) < TOL
        assert rel(tk.back_project(y, geom, True).data, g["bpw"]) < TOL
        assert rel(tk.filter_stage(y, geom, "shepp_logan").data, g["filt"]) < TOL
        assert rel(tk.fdk_cone_3d(y, geom, "shepp_logan").data, g["fdk"]) < TOL

    def test_cone_helical_and_tilted(self, tk, golden):
        g = golden("cone3d_general")
        gh = tk.GeometryCone3D((14, 18, 16), (1.1, 0.9, 1.0), (10, 14), (1.5, 1.8),
                               [tk.ProjectionMatrix(m) for m in g["mats_helix"]], 1200.0, 750.0)
        assert rel(tk.forward_project(tk.Volume(g["xh"], (1.1, 0.9, 1.0)), gh).data, g["fp_h"]) < TOL
        assert rel(tk.back_project(tk.Sinogram(g["yh"], (1.5, 1.8)), gh, True).data, g["bp_h"]) < TOL
        gt = tk.GeometryCone3D((12, 12, 12), (1, 1, 1), (12, 12), (1.6, 1.6),
                               [tk.ProjectionMatrix(m) for m in g["mats_tilt"]], 1200.0, 750.0)
        assert rel(tk.forward_project(tk.Volume(g["xt"], (1, 1, 1)), gt).data, g["fp_t"]) < TOL
        assert rel(tk.back_project(tk.Sinogram(g["yt"], (1.6, 1.6)), gt, True).data, g["bp_t"]) < TOL


# ---------------------------------------------------------------------------
# C-oracle parity at larger sizes
# ---------------------------------------------------------------------------


def cone(tk, n, det, ds, views, spacing=1.0, sdd=1200.0, sid=750.0):
    return tk.circular_cone_geometry((n, n, n), (spacing,) * 3, (det, det), (ds, ds), views, 2 * np.pi,
                                     sdd, sid)


class TestOracle:
    def test_cone_fp_bp_64(self, tk, oracle):
        geom = cone(tk, 64, 96, 1.6, 40)
        x = oracle.shepp_logan_3d((64, 64, 64)) + 0.1 * np.random.default_rng(1).standard_normal((64,) * 3)
        mats = geom.matrix_array()
        fp = tk.forward_project(tk.Volume(x, (1, 1, 1)), geom).data
        assert rel(fp, oracle.forward_cone_3d(x, (1, 1, 1), mats, (96, 96), 0.5)) < TOL
        y = np.random.default_rng(2).standard_normal((40, 96, 96))
        for w in (False, True):
            bp = tk.back_project(tk.Sinogram(y, (1.6, 1.6)), geom, w).data
            assert rel(bp, oracle.back_cone_3d(y, mats, 750.0, (64,) * 3, (1, 1, 1), w)) < TOL

    def test_fdk_128_shepp_logan(self, tk, oracle):
        # the survey's fp32 precision probe: 128^3 @1mm, 256^2 @(400/256, 600/256) mm, 180 views
        n = 128
        geom = tk.circular_cone_geometry((n,) * 3, (1, 1, 1), (256, 256), (400 / 256, 600 / 256), 180,
                                         2 * np.pi, 1200.0, 750.0)
        x = oracle.shepp_logan_3d((n,) * 3)
        mats = geom.matrix_array()
        sino = oracle.forward_cone_3d(x, (1, 1, 1), mats, (256, 256), 0.5)
        want = oracle.fdk_cone_3d(sino, mats, 1200.0, 750.0, (400 / 256, 600 / 256), (n,) * 3, (1, 1, 1),
                                  "shepp_logan")
        got = tk.fdk_cone_3d(tk.Sinogram(sino, (400 / 256, 600 / 256)), geom, "shepp_logan").data
        assert rel(got, want) < TOL
        got_fp = tk.forward_project(tk.Volume(x, (1, 1, 1)), geom).data
        assert rel(got_fp, sino) < TOL

    def test_cfg4_view_subset(self, tk, oracle):
        """Headline geometry (512^3 @0.5 mm, 1024^2 @0.6 mm) on 6 views of the 720-view
        orbit (0, 22.5, 45, 135, 202.5, 315 degrees: axis-aligned and oblique, where
        rays enter through both x and y faces), full detector resolution."""
        full = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * np.pi,
                                         1200.0, 750.0)
        mats = full.matrix_array()[[0, 45, 90, 270, 405, 630]]
        geom = tk.GeometryCone3D((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6),
                                 [tk.ProjectionMatrix(m) for m in mats], 1200.0, 750.0)
        x = tk.phantoms.shepp_logan_3d((512,) * 3)
        xh = x.cpu().numpy().astype(np.float64)
        fp = tk.forward_project(tk.Volume(x, (0.5,) * 3), geom).data
        want = oracle.forward_cone_3d(xh, (0.5,) * 3, mats, (1024, 1024), 0.25)
        assert rel(fp, want) < TOL
        filt = oracle.filter_stage_cone(want, 1200.0, 750.0, (0.6, 0.6), "shepp_logan")
        bp = tk.back_project(tk.Sinogram(filt, (0.6, 0.6)), geom, True).data
        assert rel(bp, oracle.back_cone_3d(filt, mats, 750.0, (512,) * 3, (0.5,) * 3, True)) < TOL

    def test_2d_larger(self, tk, oracle):
        ang = tk.circular_trajectory_2d(180, np.pi)
        gp = tk.GeometryParallel2D((256, 256), (1.0, 1.0), 367, 1.0, ang)
        x = np.random.default_rng(3).standard_normal((256, 256))
        assert rel(tk.forward_project(tk.Volume(x, (1, 1)), gp).data,
                   oracle.forward_parallel_2d(x, (1, 1), ang, 367, 1.0, 0.5)) < TOL
        angf = tk.circular_trajectory_2d(360, 2 * np.pi)
        gf = tk.GeometryFan2D((512, 512), (1.0, 1.0), 768, 1.6, angf, sdd=1200.0, sid=750.0)
        x = np.random.default_rng(4).standard_normal((512, 512))
        assert rel(tk.forward_project(tk.Volume(x, (1, 1)), gf).data,
                   oracle.forward_fan_2d(x, (1, 1), angf, 1200.0, 750.0, 768, 1.6, 0.5)) < TOL
        y = np.random.default_rng(5).standard_normal((360, 768))
        assert rel(tk.back_project(tk.Sinogram(y, (1.6,)), gf, True).data,
                   oracle.back_fan_2d(y, angf, 1200.0, 750.0, 1.6, (512, 512), (1, 1), True)) < TOL

    def test_edge_cases(self, tk, oracle):
        # ragged sizes, detector larger / smaller than the volume shadow, odd extents
        geom = tk.GeometryCone3D((7, 9, 5), (0.8, 1.3, 0.9), (3, 17), (2.5, 0.7),
                                 tk.circular_trajectory_3d(5, 1.3, 1200.0, 750.0, (3, 17), (2.5, 0.7)),
                                 1200.0, 750.0)
        rng = np.random.default_rng(9)
        x = rng.standard_normal((7, 9, 5))
        mats = geom.matrix_array()
        st = 0.5 * 0.8
        assert rel(tk.forward_project(tk.Volume(x, (0.8, 1.3, 0.9)), geom).data,
                   oracle.forward_cone_3d(x, (0.8, 1.3, 0.9), mats, (3, 17), st)) < TOL
        y = rng.standard_normal((5, 3, 17))
        assert rel(tk.back_project(tk.Sinogram(y, (2.5, 0.7)), geom, True).data,
                   oracle.back_cone_3d(y, mats, 750.0, (7, 9, 5), (0.8, 1.3, 0.9), True)) < TOL
        # a single view, a single detector row
        g1 = tk.circular_cone_geometry((16, 16, 16), (1, 1, 1), (1, 40), (1.0, 1.0), 1, 2 * np.pi, 1200.0, 750.0)
        x = rng.standard_normal((16, 16, 16))
        assert rel(tk.forward_project(tk.Volume(x, (1, 1, 1)), g1).data,
                   oracle.forward_cone_3d(x, (1, 1, 1), g1.matrix_array(), (1, 40), 0.5)) < TOL

    def test_zero_in_zero_out(self, tk):
        geom = cone(tk, 16, 12, 1.6, 6)
        assert not tk.forward_project(tk.Volume(np.zeros((16,) * 3), (1, 1, 1)), geom).data.any()
        assert not tk.back_project(tk.Sinogram(np.zeros((6, 12, 12)), (1.6, 1.6)), geom, True).data.any()
        assert not tk.fdk_cone_3d(tk.Sinogram(np.zeros((6, 12, 12)), (1.6, 1.6)), geom).data.any()


# ---------------------------------------------------------------------------
# analytic known-answer tests (reference test_projectors.py:64-163)
# ---------------------------------------------------------------------------


class TestChords:
    def test_cone_central_ray(self, tk):
        geom = tk.circular_cone_geometry((128,) * 3, (1, 1, 1), (25, 25), (2.0, 2.0), 1, 2 * np.pi, 1200.0, 750.0)
        ball = tk.phantoms.ball_phantom((128,) * 3, 40.0)
        sino = tk.forward_project(tk.Volume(ball, (1, 1, 1)), geom, tk.SamplingConfig(1.0)).data
        assert abs(float(sino[0, 12, 12]) - 80.0) <= 2.0

    def test_parallel_random_offsets(self, tk, rng):
        shape, sp = (256, 256), (0.5, 0.5)
        disk = tk.phantoms.disk_phantom(shape, 40.0, 1.0, sp)
        angles = rng.uniform(0, 2 * np.pi, 100)
        geom = tk.GeometryParallel2D(shape, sp, 181, 0.45, angles)
        sino = tk.forward_project(tk.Volume(disk, sp), geom, tk.SamplingConfig(1.0)).data.cpu().numpy()
        offsets = (np.arange(181) - 90) * 0.45
        js = np.clip(rng.integers(0, 160, 100) + 10, 10, 170)
        for i in range(100):
            expected = 2 * np.sqrt(max(40.0**2 - offsets[js[i]] ** 2, 0.0))
            assert abs(sino[i, js[i]] - expected) <= 1.0


# ---------------------------------------------------------------------------
# matched adjoints and autograd
# ---------------------------------------------------------------------------


class TestAdjoint:
    def test_cone_matched_dot_test(self, tk):
        geom = cone(tk, 32, 24, 2.0, 20, spacing=0.9)
        op = tk.forward_projection_op(geom, matched=True)
        assert tk.dot_test(op, trials=4) <= 1e-4
        opb = tk.back_projection_op(geom, matched=True)
        assert tk.dot_test(opb, trials=4) <= 1e-4

    def test_2d_matched_dot_test(self, tk):
        ang = tk.circular_trajectory_2d(90, 2 * np.pi)
        gp = tk.GeometryParallel2D((64, 64), (0.5, 0.5), 96, 0.8, ang)
        gf = tk.GeometryFan2D((64, 64), (1, 1), 96, 1.1, ang, sdd=1200.0, sid=750.0)
        for g in (gp, gf):
            assert tk.dot_test(tk.forward_projection_op(g, matched=True), trials=4) <= 1e-4

    def test_cfg5_full_size_matched_dot_test(self, tk):
        """The north star's adjoint test at the cfg5 size (512^3, 720 views, 1024^2,
        helical over 4 pi): <A x, y> vs <x, A^T y> for the quad-scatter transpose, on a
        smooth phantom plus noise and on white noise (float64 inner products)."""
        from paper_2511_08427_b200.projectors import fp_adjoint_tensor, fp_tensor

        mats = tk.helical_trajectory_3d(720, 4 * np.pi, 1200.0, 750.0, (1024, 1024), (0.6, 0.6), -64.0, 64.0)
        geom = tk.GeometryCone3D((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), mats, 1200.0, 750.0)
        g = torch.Generator(device="cuda").manual_seed(5)
        xs = [tk.phantoms.shepp_logan_3d((512,) * 3) + 0.1 * torch.randn((512,) * 3, device="cuda", generator=g),
              torch.randn((512,) * 3, device="cuda", generator=g)]
        for x in xs:
            y = torch.randn((720, 1024, 1024), device="cuda", generator=g)
            lhs = float((fp_tensor(x, geom, 0.25).double() * y.double()).sum())
            rhs = float((x.double() * fp_adjoint_tensor(y, geom, 0.25).double()).sum())
            assert abs(lhs - rhs) / max(abs(lhs), abs(rhs)) < 1e-4, (lhs, rhs)
            del y
            torch.cuda.empty_cache()

    def test_matched_equals_oracle_transpose(self, tk, oracle):
        geom = cone(tk, 12, 10, 1.7, 5)
        y = np.random.default_rng(11).standard_normal((5, 10, 10))
        got = tk.transpose_forward_project(tk.Sinogram(y, (1.7, 1.7)), geom).data
        want = oracle.forward_cone_3d_T(y, (12,) * 3, (1, 1, 1), geom.matrix_array(), 0.5)
        assert rel(got, want) < TOL
        x = np.random.default_rng(12).standard_normal((12,) * 3)
        got = tk.transpose_back_project(tk.Volume(x, (1, 1, 1)), geom, True).data
        want = oracle.back_cone_3d_T(x, geom.matrix_array(), 750.0, (10, 10), (1, 1, 1), True)
        assert rel(got, want) < TOL

    def test_paired_gradient_is_backprojection(self, tk):
        geom = cone(tk, 16, 12, 1.6, 8)
        x = torch.randn(16, 16, 16, device="cuda", requires_grad=True)
        y = torch.randn(8, 12, 12, device="cuda")
        (tk.ConeProjection3D.apply(x, geom) * y).sum().backward()
        want = tk.back_project(tk.Sinogram(y, (1.6, 1.6)), geom).data
        assert torch.equal(x.grad, want)

    def test_matched_gradient_and_batch(self, tk):
        geom = cone(tk, 16, 12, 1.6, 8)
        x = torch.randn(3, 16, 16, 16, device="cuda", requires_grad=True)
        y = torch.randn(3, 8, 12, 12, device="cuda")
        (tk.ConeProjection3D.apply(x, geom, "matched") * y).sum().backward()
        for i in range(3):
            want = tk.transpose_forward_project(tk.Sinogram(y[i], (1.6, 1.6)), geom).data
            assert rel(x.grad[i], want.cpu().numpy()) < 1e-5

    def test_backprojection_layer_gradient(self, tk):
        geom = cone(tk, 16, 12, 1.6, 8)
        y = torch.randn(8, 12, 12, device="cuda", requires_grad=True)
        x = torch.randn(16, 16, 16, device="cuda")
        (tk.ConeBackProjection3D.apply(y, geom) * x).sum().backward()
        assert torch.equal(y.grad, tk.forward_project(tk.Volume(x, (1, 1, 1)), geom).data)

    def test_grad_check_projectors(self, tk):
        ang = tk.circular_trajectory_2d(360, 2 * np.pi)
        g = tk.GeometryParallel2D((32, 32), (1, 1), 64, 1.0, ang)
        rep = tk.grad_check(tk.forward_projection_op(g), trials=3, epsilon=1.0)
        assert rep.passed, str(rep)
        rep = tk.grad_check(tk.forward_projection_op(g, matched=True), trials=3, epsilon=1.0, tolerance=1e-4)
        assert rep.passed, str(rep)

    def test_pyronn_listing1(self, tk):
        params = dict(volume_shape=[32, 32, 32], volume_spacing=[0.5, 0.5, 0.5], detector_shape=[40, 60],
                      detector_spacing=[1, 1], number_of_projections=36, angular_range=2 * np.pi,
                      sdd=1200, sid=750)
        geom = tk.GeometryCone3D(**params)
        geom.set_trajectory(tk.circular_trajectory_3d(**params))
        phantom = tk.phantoms.shepp_logan_3d(params["volume_shape"])[None]
        sino = tk.ConeProjectionFor3D().forward(phantom, geom)
        assert sino.shape == (1, 36, 40, 60)
        x = tk.fft_and_ifft(sino, tk.shepp_logan_3D(**params))
        reco = tk.ConeBackProjectionFor3D().forward(x, geom)
        assert reco.shape == (1, 32, 32, 32) and torch.isfinite(reco).all()


# ---------------------------------------------------------------------------
# determinism, linearity, boundary
# ---------------------------------------------------------------------------


class TestProperties:
    def test_repeat_runs_bit_identical(self, tk):
        geom = cone(tk, 32, 40, 1.6, 12)
        x = tk.Volume(np.random.default_rng(0).standard_normal((32,) * 3), (1, 1, 1))
        a = tk.forward_project(x, geom).data
        b = tk.forward_project(x, geom).data
        assert torch.equal(a, b)
        s = tk.Sinogram(a, (1.6, 1.6))
        assert torch.equal(tk.back_project(s, geom, True).data, tk.back_project(s, geom, True).data)

    def test_linearity(self, tk):
        geom = cone(tk, 16, 16, 1.6, 8)
        g = torch.Generator(device="cuda").manual_seed(0)
        x, y = (torch.randn(16, 16, 16, device="cuda", generator=g) for _ in range(2))
        step = 0.5
        from paper_2511_08427_b200.projectors import bp_tensor, fp_tensor

        lhs = fp_tensor(2.3 * x - 1.4 * y, geom, step)
        rhs = 2.3 * fp_tensor(x, geom, step) - 1.4 * fp_tensor(y, geom, step)
        assert float((lhs - rhs).abs().max()) <= 1e-5 * max(1.0, float(rhs.abs().max()))
        s, t = (torch.randn(8, 16, 16, device="cuda", generator=g) for _ in range(2))
        lhs = bp_tensor(2.3 * s - 1.4 * t, geom, True)
        rhs = 2.3 * bp_tensor(s, geom, True) - 1.4 * bp_tensor(t, geom, True)
        assert float((lhs - rhs).abs().max()) <= 1e-5 * max(1.0, float(rhs.abs().max()))

    def test_boundary_numpy_roundtrip(self, tk):
        from paper_2511_08427_b200 import ops

        cfg = {"geometry_kind": "cone3d", "volume_shape": [16, 16, 16], "volume_spacing": [1, 1, 1],
               "detector_shape": [12, 12], "detector_spacing": [1.6, 1.6], "number_of_projections": 8,
               "angular_range": 2 * np.pi, "sdd": 1200.0, "sid": 750.0}
        x = np.random.default_rng(7).standard_normal((16, 16, 16)).astype(np.float32)
        a = ops.py_forward_project(x, cfg)
        b = ops.py_forward_project(x, cfg)
        assert isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous
        assert a.shape == (8, 12, 12) and not np.shares_memory(a, b) and a.tobytes() == b.tobytes()
        with pytest.raises(ops.BoundaryError, match="float32"):
            ops.py_forward_project(x.astype(np.float64), cfg)
        pinned = torch.from_numpy(x).pin_memory()
        c = ops.py_forward_project(pinned, cfg)
        assert isinstance(c, torch.Tensor) and not c.is_cuda and c.numpy().tobytes() == a.tobytes()
        d = ops.py_forward_project(torch.from_numpy(x).cuda(), cfg)
        assert d.is_cuda and d.cpu().numpy().tobytes() == a.tobytes()
        assert ops.py_vjp_forward_project(a, cfg).tobytes() == ops.py_back_project(a, cfg).tobytes()

    def test_concurrent_calls_match_serial(self, tk):
        from concurrent.futures import ThreadPoolExecutor

        from paper_2511_08427_b200 import ops

        cfg = {"geometry_kind": "parallel2d", "volume_shape": [16, 16], "volume_spacing": [1, 1],
               "detector_shape": [24], "detector_spacing": [1.0], "number_of_projections": 12,
               "angular_range": 2 * np.pi}
        rng = np.random.default_rng(3)
        xs = [rng.standard_normal((16, 16)).astype(np.float32) for _ in range(8)]
        serial = [ops.py_forward_project(x, cfg) for x in xs]
        with ThreadPoolExecutor(max_workers=4) as pool:
            par = list(pool.map(lambda x: ops.py_forward_project(x, cfg), xs))
        assert all(s.tobytes() == p.tobytes() for s, p in zip(serial, par))

    def test_fbp_disk_fidelity(self, tk):
        shape, sp = (256, 256), (1.0, 1.0)
        disk = tk.phantoms.disk_phantom(shape, 40.0, 1.0, sp)
        geom = tk.GeometryParallel2D(shape, sp, 363, 1.0, tk.circular_trajectory_2d(360, 2 * np.pi))
        rec = tk.fbp_parallel_2d(tk.forward_project(tk.Volume(disk, sp), geom), geom, "shepp_logan").data
        y = torch.arange(256, device="cuda") - 127.5
        mask = y[None, :] ** 2 + y[:, None] ** 2 <= (0.9 * 40.0) ** 2
        rmse = float(torch.sqrt(torch.mean((rec[mask] - disk[mask]) ** 2)))
        assert rmse < 0.05

    def test_phantom_matches_oracle(self, tk, oracle):
        got = tk.phantoms.shepp_logan_3d((64, 48, 32)).cpu().numpy()
        want = oracle.shepp_logan_3d((64, 48, 32))
        assert np.mean(np.abs(got - want) > 1e-6) < 1e-4  # fp32 vs fp64 values

    def test_native_library_was_used(self, tk):
        from paper_2511_08427_b200 import _lib

        before = _lib.launch_count()
        geom = cone(tk, 16, 12, 1.6, 4)
        tk.forward_project(tk.Volume(np.ones((16,) * 3), (1, 1, 1)), geom)
        assert _lib.launch_count() > before


# ---------------------------------------------------------------------------
# every kernel variant (TK_FP_ALGO / TK_BP_ALGO) against the oracle
# ---------------------------------------------------------------------------


def _poison(shape):
    """Leave a NaN-filled block of this size in torch's caching allocator, so an output
    the next call allocates with torch.empty starts as NaN: a kernel that misses part
    of its output (e.g. a grid/CTA-shape mismatch) fails loudly instead of reading
    back a stale correct result from an earlier call."""
    t = torch.full(shape, float("nan"), device="cuda")
    del t


FP_KNOBS = [{}, {"TK_FP_MIRROR": "1"}, {"TK_FP_CFG": "4x4"}, {"TK_FP_CFG": "8x2"}, {"TK_FP_CFG": "8x1", "TK_FP_MIRROR": "1"},
            {"TK_FP_CFG": "8x2", "TK_FP_MIRROR": "1"}, {"TK_FP_CFG": "6x2", "TK_FP_MIRROR": "1"}, {"TK_FP_ALGO": "tex"},
            {"TK_FP_ALGO": "warp"}]


@pytest.mark.parametrize("knobs", FP_KNOBS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()) or "default")
def test_fp_variants_match_oracle(tk, oracle, monkeypatch, knobs):
    """Every forward-projector kernel / launch configuration against
    the oracle on circular (mirror-eligible), helical and long orbits."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    geom = tk.GeometryCone3D((24, 28, 20), (0.9, 1.1, 1.0), (30, 34), (1.5, 1.4),
                             tk.circular_trajectory_3d(17, 2 * np.pi, 1200.0, 750.0, (30, 34), (1.5, 1.4)),
                             1200.0, 750.0)
    x = np.random.default_rng(21).standard_normal((24, 28, 20))
    _poison((17, 30, 34))
    got = tk.forward_project(tk.Volume(x, (0.9, 1.1, 1.0)), geom).data
    assert bool(torch.isfinite(got).all())
    want = oracle.forward_cone_3d(x, (0.9, 1.1, 1.0), geom.matrix_array(), (30, 34), 0.45)
    assert rel(got, want) < TOL
    g = oracle  # helical trajectory (non-circular orbit)
    hel = tk.helical_trajectory_3d(13, 4 * np.pi, 1200.0, 750.0, (30, 34), (1.5, 1.4), -8.0, 8.0)
    gh = tk.GeometryCone3D((24, 28, 20), (0.9, 1.1, 1.0), (30, 34), (1.5, 1.4), hel, 1200.0, 750.0)
    _poison((13, 30, 34))
    got = tk.forward_project(tk.Volume(x, (0.9, 1.1, 1.0)), gh).data
    assert bool(torch.isfinite(got).all())
    want = g.forward_cone_3d(x, (0.9, 1.1, 1.0), gh.matrix_array(), (30, 34), 0.45)
    assert rel(got, want) < TOL
    # a long orbit (>= 128 views: 8 views per CTA in the default kernel)
    gl = tk.circular_cone_geometry((24, 28, 20), (0.9, 1.1, 1.0), (30, 34), (1.5, 1.4), 131, 2 * np.pi,
                                   1200.0, 750.0)
    _poison((131, 30, 34))
    got = tk.forward_project(tk.Volume(x, (0.9, 1.1, 1.0)), gl).data
    assert bool(torch.isfinite(got).all())
    assert rel(got, g.forward_cone_3d(x, (0.9, 1.1, 1.0), gl.matrix_array(), (30, 34), 0.45)) < TOL


@pytest.mark.parametrize("knobs", [{}, {"TK_FPT_CARRY": "0"}])
def test_fp_transpose_matches_oracle(tk, oracle, monkeypatch, knobs):
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    shape, sp = (20, 26, 22), (1.1, 0.9, 1.0)
    hel = tk.helical_trajectory_3d(11, 4 * np.pi, 1200.0, 750.0, (30, 34), (1.5, 1.4), -8.0, 8.0)
    for mats in (hel, tk.circular_trajectory_3d(13, 2 * np.pi, 1200.0, 750.0, (30, 34), (1.5, 1.4))):
        geom = tk.GeometryCone3D(shape, sp, (30, 34), (1.5, 1.4), mats, 1200.0, 750.0)
        y = np.random.default_rng(31).standard_normal((len(mats), 30, 34))
        got = tk.transpose_forward_project(tk.Sinogram(y, (1.5, 1.4)), geom).data
        want = oracle.forward_cone_3d_T(y, shape, sp, geom.matrix_array(), 0.45)
        assert rel(got, want) < TOL


def test_2d_bp_transpose_matches_oracle(tk, oracle):
    """Exact B^T of the 2D voxel-driven back projectors (parallel; fan with and without
    the distance weight) against the oracle's transposes, plus the matched dot test
    and the autograd path BackProjection(adjoint='matched')."""
    rng = np.random.default_rng(41)
    ang = tk.circular_trajectory_2d(53, np.pi)
    gp = tk.GeometryParallel2D((37, 41), (0.9, 1.1), 59, 1.3, ang)
    x = rng.standard_normal((37, 41))
    got = tk.transpose_back_project(tk.Volume(x, (0.9, 1.1)), gp).data
    assert rel(got, oracle.back_parallel_2d_T(x, ang, 1.3, 59, (0.9, 1.1))) < TOL
    angf = tk.circular_trajectory_2d(61, 2 * np.pi)
    gf = tk.GeometryFan2D((37, 41), (0.9, 1.1), 70, 1.6, angf, sdd=1200.0, sid=750.0)
    for w in (False, True):
        got = tk.transpose_back_project(tk.Volume(x, (0.9, 1.1)), gf, w).data
        assert rel(got, oracle.back_fan_2d_T(x, angf, 1200.0, 750.0, 1.6, 70, (0.9, 1.1), w)) < TOL
    for g in (gp, gf):
        assert tk.dot_test(tk.back_projection_op(g, matched=True), trials=3) <= 1e-4
    # wide detector: global-atomic path (rows longer than the shared-memory row buffer);
    # detector coordinates are formed relative to the centre, so fp32 keeps the
    # interpolation weights accurate 6500 pixels out
    gw = tk.GeometryParallel2D((24, 24), (1.0, 1.0), 13000, 0.01, ang[:5])
    xw = rng.standard_normal((24, 24))
    got = tk.transpose_back_project(tk.Volume(xw, (1.0, 1.0)), gw).data
    assert rel(got, oracle.back_parallel_2d_T(xw, ang[:5], 0.01, 13000, (1.0, 1.0))) < TOL
    yw = rng.standard_normal((5, 13000))
    got = tk.back_project(tk.Sinogram(yw, (0.01,)), gw).data
    assert rel(got, oracle.back_parallel_2d(yw, ang[:5], 0.01, (24, 24), (1.0, 1.0))) < TOL
    y = torch.tensor(rng.standard_normal((61, 70)), dtype=torch.float32, device="cuda", requires_grad=True)
    out = tk.FanBackProjection2D.apply(y, gf, "matched", True)
    gx = torch.randn_like(out)
    out.backward(gx)
    want = tk.transpose_back_project(tk.Volume(gx, (0.9, 1.1)), gf, True).data
    assert rel(y.grad, want.cpu().numpy()) < 1e-6


def test_bp_transpose_matches_oracle(tk, oracle):
    shape, sp = (20, 26, 22), (1.1, 0.9, 1.0)
    hel = tk.helical_trajectory_3d(11, 4 * np.pi, 1200.0, 750.0, (30, 34), (1.5, 1.4), -8.0, 8.0)
    x = np.random.default_rng(32).standard_normal(shape)
    for mats in (hel, tk.circular_trajectory_3d(13, 2 * np.pi, 1200.0, 750.0, (30, 34), (1.5, 1.4))):
        geom = tk.GeometryCone3D(shape, sp, (30, 34), (1.5, 1.4), mats, 1200.0, 750.0)
        for w in (False, True):
            got = tk.transpose_back_project(tk.Volume(x, sp), geom, w).data
            want = oracle.back_cone_3d_T(x, geom.matrix_array(), 750.0, (30, 34), sp, w)
            assert rel(got, want) < TOL


@pytest.mark.parametrize("algo", ["tma", "quad", "tex"])
def test_bp_variants_match_oracle(tk, oracle, golden, monkeypatch, algo):
    monkeypatch.setenv("TK_BP_ALGO", algo)
    geom = cone(tk, 24, 36, 1.5, 19)
    y = np.random.default_rng(22).standard_normal((19, 36, 36))
    for w in (False, True):
        got = tk.back_project(tk.Sinogram(y, (1.5, 1.5)), geom, w).data
        assert rel(got, oracle.back_cone_3d(y, geom.matrix_array(), 750.0, (24,) * 3, (1, 1, 1), w)) < TOL
    g = golden("cone3d_general")  # tilted detector: general (z-varying) path
    gt = tk.GeometryCone3D((12, 12, 12), (1, 1, 1), (12, 12), (1.6, 1.6),
                           [tk.ProjectionMatrix(m) for m in g["mats_tilt"]], 1200.0, 750.0)
    assert rel(tk.back_project(tk.Sinogram(g["yt"], (1.6, 1.6)), gt, True).data, g["bp_t"]) < TOL


@pytest.mark.parametrize("algo", ["tma", "quad", "tex"])
def test_bp_row_band_zslab(tk, oracle, monkeypatch, algo):
    """Sharded building block: a z-slab from a cropped detector row band equals
    the same slab of the full back projection."""
    monkeypatch.setenv("TK_BP_ALGO", algo)
    from paper_2511_08427_b200 import distributed as D
    from paper_2511_08427_b200.projectors import bp_cone_tensor_ex

    geom = tk.circular_cone_geometry((32, 24, 20), (1.0, 1.0, 1.0), (48, 40), (1.5, 1.5), 12, 2 * np.pi,
                                     1200.0, 750.0)
    y = torch.randn(12, 48, 40, device="cuda")
    full = tk.back_project(tk.Sinogram(y, (1.5, 1.5)), geom, True).data
    for world in (2, 3):
        for rank in range(world):
            z0, z1 = D.shard_bounds(32, world, rank)
            r0, r1 = D.row_band(geom, z0, z1)
            slab = bp_cone_tensor_ex(y[:, r0:r1].contiguous(), geom, True, r0, z0, z1 - z0)
            assert rel(slab, full[z0:z1].cpu().numpy()) < 1e-5  # fp32 row-shift rounding


@pytest.mark.parametrize("algo", ["tma"])
@pytest.mark.parametrize("det_pitch", [0.05, 0.4, 3.0])
def test_bp_tile_rectangles_and_fallback(tk, oracle, monkeypatch, det_pitch, algo):
    """Fine detector pitch makes the CTA footprint exceed the shared-memory tile
    (global-gather fallback); coarse pitch makes whole volumes fit one tile."""
    monkeypatch.setenv("TK_BP_ALGO", algo)
    geom = tk.circular_cone_geometry((20, 36, 33), (1.0, 0.8, 1.2), (40, 50), (det_pitch, det_pitch), 7,
                                     2 * np.pi, 1200.0, 750.0)
    y = np.random.default_rng(23).standard_normal((7, 40, 50))
    got = tk.back_project(tk.Sinogram(y, (det_pitch, det_pitch)), geom, True).data
    want = oracle.back_cone_3d(y, geom.matrix_array(), 750.0, (20, 36, 33), (1.0, 0.8, 1.2), True)
    assert rel(got, want) < TOL


def test_overlapped_host_pipeline_matches_device(tk):
    """Pinned-host boundary calls (chunked plan projection with overlapped D2H,
    chunked H2D + filtering + accumulating back projection) equal the
    device-resident operators (bit for bit for the projection; to summation
    order for the chunked FDK)."""
    from paper_2511_08427_b200 import ops
    from paper_2511_08427_b200.filters import fdk_tensor
    from paper_2511_08427_b200.projectors import ForwardProjectionPlan, fp_tensor

    cfg = {"geometry_kind": "cone3d", "volume_shape": [40, 48, 44], "volume_spacing": [1.0, 1.0, 1.0],
           "detector_shape": [50, 60], "detector_spacing": [1.4, 1.4], "number_of_projections": 37,
           "angular_range": 2 * np.pi, "sdd": 1200.0, "sid": 750.0, "filter_kind": "cosine"}
    geom = ops.PipelineConfig.from_dict(cfg).build_geometry()
    x = torch.randn(40, 48, 44)
    want = fp_tensor(x.cuda(), geom, 0.5)
    got = ops.py_forward_project(x.pin_memory(), cfg)
    assert got.is_pinned() and torch.equal(got, want.cpu())
    with ForwardProjectionPlan(x.cuda(), geom) as plan:
        part = torch.empty(10, 50, 60, device="cuda")
        plan.project(slice(5, 15), part, 0.5)
        assert torch.equal(part, want[5:15])
    rec = ops.py_fbp(got, cfg)  # view-chunked filter + accumulating back projection
    assert rec.is_pinned() and rel(rec, fdk_tensor(want, geom, "cosine").cpu()) < 1e-6


def test_grid_files_roundtrip_and_reference_format(tk, tmp_path, golden):
    """Grid pairs written here read back bit-exactly and carry the reference's
    header schema (grids.py:122-212)."""
    import json

    x = golden("cone3d")["x"]
    v = tk.Volume(x, (1.0, 1.0, 1.0))
    tk.write_grid(v, tmp_path / "vol")
    hdr = json.loads((tmp_path / "vol.json").read_text())
    assert hdr == {"kind": "volume", "shape": [16, 16, 16], "spacing": [1.0, 1.0, 1.0], "dtype": "f32le",
                   "order": "C"}
    back = tk.read_grid(tmp_path / "vol.raw")
    assert torch.equal(back.data, v.data)
    s = tk.Sinogram(golden("cone3d")["y"], (1.6, 1.6))
    tk.write_grid(s, tmp_path / "sino.json")
    s2 = tk.read_grid(tmp_path / "sino")
    assert isinstance(s2, tk.Sinogram) and s2.detector_spacing == (1.6, 1.6) and torch.equal(s2.data, s.data)
    with pytest.raises(tk.SizeMismatchError):
        (tmp_path / "bad.json").write_text((tmp_path / "vol.json").read_text())
        (tmp_path / "bad.raw").write_bytes(b"\0" * 12)
        tk.read_grid(tmp_path / "bad")


def test_2d_layers_autograd(tk):
    ang = tk.circular_trajectory_2d(60, 2 * np.pi)
    gp = tk.GeometryParallel2D((24, 24), (1, 1), 36, 1.0, ang)
    gf = tk.GeometryFan2D((24, 24), (1, 1), 40, 1.5, ang, sdd=1200.0, sid=750.0)
    for fwd, bwd, g in ((tk.ParallelProjection2D, tk.ParallelBackProjection2D, gp),
                        (tk.FanProjection2D, tk.FanBackProjection2D, gf)):
        x = torch.randn(24, 24, device="cuda", requires_grad=True)
        y = torch.randn(*g.sinogram_shape, device="cuda")
        (fwd.apply(x, g) * y).sum().backward()
        assert torch.equal(x.grad, tk.back_project(tk.Sinogram(y, (g.detector_spacing,)), g).data)
        x2 = torch.randn(24, 24, device="cuda", requires_grad=True)
        (fwd.apply(x2, g, "matched") * y).sum().backward()
        want = tk.transpose_forward_project(tk.Sinogram(y, (g.detector_spacing,)), g).data
        assert rel(x2.grad, want.cpu().numpy()) < 1e-5
        s = torch.randn(*g.sinogram_shape, device="cuda", requires_grad=True)
        xx = torch.randn(24, 24, device="cuda")
        (bwd.apply(s, g) * xx).sum().backward()
        assert torch.equal(s.grad, tk.forward_project(tk.Volume(xx, (1, 1)), g).data)


def test_helical_learned_reconstruction_gradient_step(tk):
    """cfg5 pattern at small scale: loss 1/2 |A x - y|^2 on a helical orbit,
    gradient through ConeProjection3D (paired and matched), one descent step
    lowers the loss."""
    mats = tk.helical_trajectory_3d(48, 4 * np.pi, 1200.0, 750.0, (40, 40), (1.2, 1.2), -8.0, 8.0)
    geom = tk.GeometryCone3D((32, 32, 32), (1, 1, 1), (40, 40), (1.2, 1.2), mats, 1200.0, 750.0)
    truth = tk.phantoms.shepp_logan_3d((32, 32, 32))
    y = tk.ConeProjection3D.apply(truth, geom) + 0.01 * torch.randn(48, 40, 40, device="cuda")
    for adjoint in ("paired", "matched"):
        x = torch.zeros(32, 32, 32, device="cuda", requires_grad=True)
        loss = 0.5 * ((tk.ConeProjection3D.apply(x, geom, adjoint) - y) ** 2).sum()
        loss.backward()
        with torch.no_grad():
            g = x.grad
            ag = tk.ConeProjection3D.apply(g, geom)
            t = float((g * g).sum() / (ag * ag).sum())  # exact line search for the matched gradient
            x2 = x - t * g
            loss2 = 0.5 * ((tk.ConeProjection3D.apply(x2, geom) - y) ** 2).sum()
        assert float(loss2) < float(loss)


@pytest.mark.parametrize("algo", ["r16", "stockham", "warp"])
@pytest.mark.parametrize("cols,rows,views", [(7, 3, 2), (200, 5, 3), (256, 9, 2), (300, 4, 3), (513, 3, 2),
                                             (1024, 6, 3), (2047, 2, 1), (3000, 2, 1)])
def test_filter_variants_match_oracle(tk, oracle, monkeypatch, algo, cols, rows, views):
    """Every row-filter kernel (TK_FILTER_ALGO) against numpy's rfft/irfft oracle,
    n_pad from 16 to 8192, odd pair counts, cone pre-weight and a row band."""
    monkeypatch.setenv("TK_FILTER_ALGO", algo)
    geom = tk.circular_cone_geometry((8, 8, 8), (1.0, 1.0, 1.0), (rows, cols), (0.7, 0.55), views,
                                     2 * np.pi, 1200.0, 750.0)
    y = np.random.default_rng(cols).standard_normal((views, rows, cols))
    got = tk.filter_stage(tk.Sinogram(T(y), (0.7, 0.55)), geom, "shepp_logan").data
    want = oracle.filter_stage_cone(y, 1200.0, 750.0, (0.7, 0.55), "shepp_logan")
    assert rel(got, want) < TOL
    from paper_2511_08427_b200.filters import filter_stage_tensor

    if rows > 2:  # band of detector rows [1, rows-1) with the global row offset
        band = filter_stage_tensor(T(y[:, 1:rows - 1]).contiguous(), geom, "shepp_logan", row_offset=1)
        assert rel(band, want[:, 1:rows - 1]) < TOL


@pytest.mark.parametrize("cols", [64, 66])
def test_bp_tma_large_volume_edges(tk, oracle, monkeypatch, cols):
    """TMA-staged back projection on a volume whose blocks reach the detector
    edges (out-of-detector texels zero-filled by the TMA unit) and a partial
    last block in every axis; cols = 66 takes the quad fallback (16-byte row pitch)."""
    monkeypatch.setenv("TK_BP_ALGO", "tma")
    geom = tk.circular_cone_geometry((37, 45, 41), (1.1, 1.0, 0.9), (40, cols), (1.3, 1.2), 23, 2 * np.pi,
                                     1200.0, 750.0)
    y = np.random.default_rng(cols).standard_normal((23, 40, cols))
    for w in (False, True):
        got = tk.back_project(tk.Sinogram(y, (1.3, 1.2)), geom, w).data
        want = oracle.back_cone_3d(y, geom.matrix_array(), 750.0, (37, 45, 41), (1.1, 1.0, 0.9), w)
        assert rel(got, want) < TOL


def test_fp_fixed_row_stride_layout_matches_runtime_stride(tk, monkeypatch):
    """Large non-cubic volume: the compile-time row-stride cell layout (immediate-offset
    far-row loads, used when it wastes at most 2x the compact layout's memory) gives
    bit-identical projections to the runtime-stride layout, views at 0/30/45/60/90
    degrees, for the general and the mirror-pair kernel."""
    shape, sp = (520, 500, 510), (0.5, 0.5, 0.5)
    full = tk.circular_cone_geometry(shape, sp, (256, 300), (2.0, 2.0), 720, 2 * np.pi, 1200.0, 750.0)
    geom = tk.GeometryCone3D(shape, sp, (256, 300), (2.0, 2.0), [full.matrices[i] for i in (0, 60, 90, 120, 180)],
                             1200.0, 750.0)
    x = torch.rand(shape, device="cuda")
    for mirror in ("0", "1"):
        monkeypatch.setenv("TK_FP_MIRROR", mirror)
        monkeypatch.setenv("TK_FP_NOFIX", "0")
        a = tk.forward_project(tk.Volume(x, sp), geom).data
        monkeypatch.setenv("TK_FP_NOFIX", "1")
        b = tk.forward_project(tk.Volume(x, sp), geom).data
        assert torch.equal(a, b) and float(a.abs().max()) > 0


def test_deterministic_cone_transpose(tk, oracle):
    """Fixed-point A^T: matches the oracle's exact transpose, is bit-identical across
    runs, and agrees with the fp32-atomic transpose to rounding."""
    from paper_2511_08427_b200.projectors import fp_adjoint_tensor

    shape, sp = (20, 26, 22), (1.1, 0.9, 1.0)
    hel = tk.helical_trajectory_3d(11, 4 * np.pi, 1200.0, 750.0, (30, 34), (1.5, 1.4), -8.0, 8.0)
    geom = tk.GeometryCone3D(shape, sp, (30, 34), (1.5, 1.4), hel, 1200.0, 750.0)
    y = np.random.default_rng(33).standard_normal((11, 30, 34))
    yt = T(y)
    a = fp_adjoint_tensor(yt, geom, 0.45, deterministic=True)
    b = fp_adjoint_tensor(yt, geom, 0.45, deterministic=True)
    assert torch.equal(a, b)
    assert rel(a, oracle.forward_cone_3d_T(y, shape, sp, geom.matrix_array(), 0.45)) < TOL
    assert rel(a, fp_adjoint_tensor(yt, geom, 0.45, deterministic=False).cpu().numpy()) < 1e-6
    assert float(fp_adjoint_tensor(torch.zeros_like(yt), geom, 0.45, deterministic=True).abs().max()) == 0.0
    torch.use_deterministic_algorithms(True)
    try:
        c = fp_adjoint_tensor(yt, geom, 0.45)  # follows torch's determinism switch
    finally:
        torch.use_deterministic_algorithms(False)
    assert torch.equal(a, c)


def test_deterministic_transpose_many_rays_per_cell(tk, oracle):
    """A detector far finer than the voxel grid (hundreds of rays per cell per
    view) with a same-sign sinogram: the fixed-point scale comes from the
    geometry's tap-contribution bound, so the int64 sums cannot wrap."""
    from paper_2511_08427_b200.projectors import fp_adjoint_tensor

    shape, sp = (6, 6, 6), (4.0, 4.0, 4.0)
    geom = cone(tk, 6, 160, 0.25, 7, spacing=4.0)
    y = np.ones((7, 160, 160))
    a = fp_adjoint_tensor(T(y), geom, 0.5, deterministic=True)
    want = oracle.forward_cone_3d_T(y, shape, sp, geom.matrix_array(), 0.5)
    assert float(a.min()) >= 0.0
    assert rel(a, want) < TOL


def test_nondeterministic_transposes_follow_torch_determinism(tk):
    """Under torch.use_deterministic_algorithms(True) the atomic-only transposes raise
    (torch's convention), warn with warn_only=True, and the cone A^T switches to its
    fixed-point form."""
    from paper_2511_08427_b200.projectors import bp_adjoint_tensor, fp_adjoint_tensor

    geom = cone(tk, 12, 10, 1.7, 5)
    x = torch.rand(12, 12, 12, device="cuda")
    y = torch.rand(5, 10, 10, device="cuda")
    torch.use_deterministic_algorithms(True)
    try:
        with pytest.raises(RuntimeError, match="deterministic"):
            bp_adjoint_tensor(x, geom)
        assert torch.equal(fp_adjoint_tensor(y, geom, 0.5), fp_adjoint_tensor(y, geom, 0.5, deterministic=True))
        torch.use_deterministic_algorithms(True, warn_only=True)
        with pytest.warns(UserWarning):
            bp_adjoint_tensor(x, geom)
    finally:
        torch.use_deterministic_algorithms(False)
    bp_adjoint_tensor(x, geom)  # fine when the switch is off


@pytest.mark.parametrize("knobs", [{"TK_FP_CFG": "4x4"}, {"TK_FP_CFG": "8x2"}, {"TK_FP_ZP": "0"}, {"TK_FP_UNR": "2"},
                                   {"TK_FP_NOFIX": "1"},
                                   {"TK_FP_MIRROR": "1"}, {"TK_FP_MIRROR": "1", "TK_FP_NOFIX": "1"},
                                   {"TK_FP_MIRROR": "1", "TK_FP_CFG": "8x1"}, {"TK_FP_MIRROR": "1", "TK_FP_CFG": "8x2"}])
def test_fp_tuning_knobs_keep_results(tk, monkeypatch, knobs):
    """Every forward-projector tuning knob (kernel, CTA shape, fixed stride) must give the default's projection (same taps; bit-identical or
    rounding-level), with no output element missed."""
    geom = tk.circular_cone_geometry((24, 28, 20), (0.9, 1.1, 1.0), (30, 34), (1.5, 1.4), 131, 2 * np.pi,
                                     1200.0, 750.0)
    x = torch.rand(24, 28, 20, device="cuda")
    want = tk.forward_project(tk.Volume(x, (0.9, 1.1, 1.0)), geom).data.clone()
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    _poison((131, 30, 34))
    got = tk.forward_project(tk.Volume(x, (0.9, 1.1, 1.0)), geom).data
    assert bool(torch.isfinite(got).all())
    assert rel(got, want.cpu().numpy()) < 1e-6


@pytest.mark.parametrize("det_pitch", [2.4, 1.5, 0.9, 0.5, 0.3])
def test_bp_tma_tile_pitches(tk, monkeypatch, det_pitch):
    """TMA back projector across detector pitches that select different compile-time tile
    pitches (44 ... 244 floats): same result as the quad back projector on a ragged
    volume, no voxel missed."""
    geom = tk.circular_cone_geometry((37, 45, 41), (1.0, 0.9, 1.1), (90, 132), (det_pitch, det_pitch), 33,
                                     2 * np.pi, 1200.0, 750.0)
    y = torch.rand(33, 90, 132, device="cuda")
    monkeypatch.setenv("TK_BP_ALGO", "quad")
    want = tk.back_project(tk.Sinogram(y, (det_pitch, det_pitch)), geom, True).data.clone()
    monkeypatch.setenv("TK_BP_ALGO", "tma")
    _poison((37, 45, 41))
    got = tk.back_project(tk.Sinogram(y, (det_pitch, det_pitch)), geom, True).data
    assert bool(torch.isfinite(got).all())
    assert rel(got, want.cpu().numpy()) < 1e-5


# ---------------------------------------------------------------------------
# z-mirror-pair forward projector (circular orbits)
# ---------------------------------------------------------------------------


class TestMirrorForward:
    @pytest.mark.parametrize("shape,spacing,det,ds,views", [
        ((64, 64, 64), (1.0, 1.0, 1.0), (96, 96), (1.6, 1.6), 40),        # even rows
        ((33, 40, 21), (0.8, 1.1, 0.9), (31, 45), (1.9, 1.4), 17),        # odd rows / odd nz, ragged
        ((20, 16, 16), (1.0, 1.0, 1.0), (7, 40), (2.5, 1.2), 9),          # detector narrower than the shadow
        ((16, 16, 16), (1.0, 1.0, 1.0), (1, 24), (1.6, 1.6), 5),          # single (middle) row
    ])
    def test_matches_oracle_and_general_kernel(self, tk, oracle, monkeypatch, shape, spacing, det, ds, views):
        from paper_2511_08427_b200.projectors import forward_kernel_path

        geom = tk.circular_cone_geometry(shape, spacing, det, ds, views, 2 * np.pi, 1200.0, 750.0)
        monkeypatch.setenv("TK_FP_MIRROR", "1")
        assert forward_kernel_path(geom) == "mirror"
        x = np.random.default_rng(7).standard_normal(shape).astype(np.float32).astype(np.float64)
        got = tk.forward_project(tk.Volume(x, spacing), geom).data
        want = oracle.forward_cone_3d(x, spacing, geom.matrix_array(), det, 0.5 * min(spacing))
        assert rel(got, want) < TOL
        monkeypatch.setenv("TK_FP_MIRROR", "0")
        general = tk.forward_project(tk.Volume(x, spacing), geom).data
        assert rel(got, general.cpu().numpy()) < 2e-6
        # the direct rows are the general kernel's rays bit for bit (same cells, same arithmetic)
        half = det[0] // 2
        assert torch.equal(got[:, :half], general[:, :half])

    @pytest.mark.parametrize("cfg", ["4x3", "8x1", "8x2"])
    def test_launch_configurations(self, tk, oracle, monkeypatch, cfg):
        monkeypatch.setenv("TK_FP_MIRROR", "1")
        monkeypatch.setenv("TK_FP_CFG", cfg)
        geom = tk.circular_cone_geometry((48,) * 3, (1.0,) * 3, (64, 80), (1.6, 1.6), 19, 2 * np.pi, 1200.0, 750.0)
        x = oracle.shepp_logan_3d((48,) * 3)
        got = tk.forward_project(tk.Volume(x, (1, 1, 1)), geom).data
        assert rel(got, oracle.forward_cone_3d(x, (1, 1, 1), geom.matrix_array(), (64, 80), 0.5)) < TOL



def test_more_views_than_a_grid_dimension(tk, oracle):
    """A helical scan with more views than 65535 (the limit of a grid's y / z dimension):
    forward projection, its transpose and both back projectors take any view count."""
    from paper_2511_08427_b200.projectors import bp_adjoint_tensor, fp_adjoint_tensor

    n_views = 70000
    mats = tk.helical_trajectory_3d(n_views, 200 * np.pi, 1200.0, 750.0, (4, 4), (8.0, 8.0), -6.0, 6.0)
    geom = tk.GeometryCone3D((8, 8, 8), (1.0, 1.0, 1.0), (4, 4), (8.0, 8.0), mats, 1200.0, 750.0)
    x = np.random.default_rng(51).standard_normal((8, 8, 8))
    got = tk.forward_project(tk.Volume(x, (1, 1, 1)), geom).data
    idx = np.array([0, 1, 65534, 65535, 65536, n_views - 1])
    sub = tk.GeometryCone3D((8, 8, 8), (1.0, 1.0, 1.0), (4, 4), (8.0, 8.0), [mats[i] for i in idx], 1200.0, 750.0)
    want = oracle.forward_cone_3d(x, (1, 1, 1), sub.matrix_array(), (4, 4), 0.5)
    assert rel(got[idx], want) < TOL
    gen = torch.Generator(device="cuda").manual_seed(52)
    y = torch.randn(geom.sinogram_shape, device="cuda", generator=gen)
    for w in (False, True):
        bp = tk.back_project(tk.Sinogram(y, (8.0, 8.0)), geom, w).data
        assert bool(torch.isfinite(bp).all()) and float(bp.abs().max()) > 0
    xt = torch.randn(8, 8, 8, device="cuda", generator=gen)
    # dot tests of both exact transposes across the whole 70000-view stack
    ax = tk.forward_project(tk.Volume(xt, (1, 1, 1)), geom).data
    at = fp_adjoint_tensor(y, geom, 0.5)
    lhs, rhs = float((ax.double() * y.double()).sum()), float((xt.double() * at.double()).sum())
    assert abs(lhs - rhs) <= 1e-4 * abs(lhs)
    # B^T on non-negative inputs: with signed inputs the 512-term dot cancels ~100x and the
    # check measures fp32 summation over 70000 views, not the transpose
    yp = torch.rand(geom.sinogram_shape, device="cuda", generator=gen)
    xp = torch.rand(8, 8, 8, device="cuda", generator=gen)
    bx = tk.back_project(tk.Sinogram(yp, (8.0, 8.0)), geom).data
    bt = bp_adjoint_tensor(xp, geom)
    lhs, rhs = float((bx.double() * xp.double()).sum()), float((yp.double() * bt.double()).sum())
    assert abs(lhs - rhs) <= 1e-4 * abs(lhs)


class TestBandRoutedForward:
    """tk_forward_cone_3d_bands: the forward kernel storing every ray straight into the
    row-band buffers of the ranks whose z-slab needs it (the fused multi-GPU exchange).
    World sizes 2..5 are simulated on one GPU with local buffers in place of peer
    addresses: the kernel does not distinguish them."""

    @pytest.mark.parametrize("world", [2, 3, 5])
    def test_bands_equal_crops_of_the_full_projection(self, tk, world):
        from paper_2511_08427_b200 import distributed as D
        from paper_2511_08427_b200.projectors import fp_bands_tensor, fp_tensor

        geom = tk.circular_cone_geometry((40, 44, 36), (1.0, 0.9, 1.1), (70, 52), (1.6, 1.5), 29, 2 * np.pi,
                                         1200.0, 750.0)
        x = torch.rand(geom.volume_shape, device="cuda")
        full = fp_tensor(x, geom, 0.5)
        bands = D.slab_bands(geom, world)
        pitch = max(r1 - r0 for (_, _, r0, r1) in bands)
        bufs = [torch.full((29, pitch, 52), float("nan"), device="cuda") for _ in range(world)]
        for g in range(world):  # every "rank" projects its view block into all bands
            vb, ve = D.shard_bounds(29, world, g)
            fp_bands_tensor(x, D.subset_geometry(geom, slice(vb, ve)), 0.5, vb, bufs,
                            [(r0, r1) for (_, _, r0, r1) in bands], pitch)
        for h, (_, _, r0, r1) in enumerate(bands):
            assert torch.equal(bufs[h][:, : r1 - r0], full[:, r0:r1]), h
            assert bool(torch.isnan(bufs[h][:, r1 - r0:]).all())  # rows beyond the band untouched

    def test_p2p_host_path_single_rank(self, tk):
        """forward_project_p2p on a 1-rank NCCL group: symmetric-memory buffer,
        rendezvous, band-routed kernel, device barriers."""
        import os

        import torch.distributed as dist

        from paper_2511_08427_b200 import distributed as D
        from paper_2511_08427_b200.projectors import fp_tensor

        if dist.is_initialized():
            pytest.skip("a process group already exists")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        try:
            geom = tk.circular_cone_geometry((32, 32, 32), (1.0,) * 3, (40, 48), (1.6, 1.6), 17, 2 * np.pi,
                                             1200.0, 750.0)
            x = torch.rand(geom.volume_shape, device="cuda")
            try:
                band = D.forward_project_p2p(x, geom, 0.5, 0, 1)
            except (RuntimeError, NotImplementedError) as exc:  # no symmetric-memory backend on this box
                pytest.skip(f"symmetric memory unavailable: {exc}")
            torch.cuda.synchronize()
            assert torch.equal(band, fp_tensor(x, geom, 0.5))
            band2 = D.forward_project_p2p(x * 2, geom, 0.5, 0, 1)  # cached buffer, second call
            assert torch.equal(band2, fp_tensor(x * 2, geom, 0.5))
        finally:
            D._symm_cache.clear()
            dist.destroy_process_group()
