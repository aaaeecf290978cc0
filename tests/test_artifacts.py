"""Sinogram degradation simulators (reference artifacts.py, tests/test_artifacts.py):
the deterministic ones against golden fixtures the reference produced
(tests/golden/make_golden_artifacts.py), the random ones against the reference's
statistical contract; the GPU path runs through libtkb200 (no CPU fallback)."""

import numpy as np
import pytest
import torch


def test_line_kernels_match_reference(golden):
    """Host-side kernel rasterisation (artifacts.py:158-180) equals the reference's."""
    from paper_2511_08427_b200.artifacts import line_kernel

    g = golden("artifacts")
    thetas = {f"{t:.4f}": t for t in (0.0, 0.3, np.pi / 4, 2.0, -1.1)}  # make_golden_artifacts.py
    keys = [k for k in g if k.startswith("kernel_")]
    assert len(keys) == 15
    for key in keys:
        _, length, theta = key.split("_")
        np.testing.assert_allclose(line_kernel(int(length), thetas[theta]), g[key], rtol=0, atol=1e-15)


@pytest.fixture(scope="module")
def tk(cuda):
    import paper_2511_08427_b200 as tk

    return tk


def sino2d(rng, n=16, w=40):
    import paper_2511_08427_b200 as tk

    return tk.Sinogram(rng.uniform(0.0, 3.0, (n, w)), (1.0,))


def sino3d(rng, n=6, rows=20, cols=24):
    import paper_2511_08427_b200 as tk

    return tk.Sinogram(rng.uniform(0.0, 3.0, (n, rows, cols)), (1.0, 1.0))


def host(s):
    return s.data.cpu().numpy().astype(np.float64)


@pytest.mark.gpu
class TestDeterministicAgainstReference:
    def test_gantry_blur(self, tk, golden):
        g = golden("artifacts")
        geom = tk.circular_cone_geometry((16, 16, 16), (1, 1, 1), (20, 24), (1.0, 1.0), 8, 2 * np.pi, 1200.0, 750.0)
        s3 = tk.Sinogram(g["sino3"], (1.0, 1.0))
        for n in (5, 9):
            out = tk.add_gantry_motion_blur(s3, geom, n)
            np.testing.assert_allclose(host(out), g[f"blur3_len{n}"], rtol=1e-5, atol=1e-6)
        g2 = tk.GeometryParallel2D((16, 16), (1, 1), 40, 1.0, tk.circular_trajectory_2d(16, 2 * np.pi))
        out2 = tk.add_gantry_motion_blur(tk.Sinogram(g["sino2"], (1.0,)), g2, 3)
        np.testing.assert_allclose(host(out2), g["blur2_len3"], rtol=1e-5, atol=1e-6)

    def test_ring(self, tk, golden):
        g = golden("artifacts")
        s3 = tk.Sinogram(g["sino3"], (1.0, 1.0))
        a = tk.add_ring_artifact(s3, [4, 17], (2, 6), "zero")
        b = tk.add_ring_artifact(s3, [0, 23], None, "scale", 0.7)
        np.testing.assert_array_equal(host(a), g["ring3_zero"].astype(np.float32))
        np.testing.assert_allclose(host(b), g["ring3_scale"], rtol=1e-6)


@pytest.mark.gpu
class TestDetectorJitter:
    def test_zero_shift_is_identity(self, tk, rng):
        s = sino2d(rng)
        assert torch.equal(tk.add_detector_jitter(s, 0, "u", seed=5).data, s.data)

    def test_same_seed_identical(self, tk, rng):
        s = sino3d(rng)
        a = tk.add_detector_jitter(s, 3, "v", seed=42)
        b = tk.add_detector_jitter(s, 3, "v", seed=42)
        assert torch.equal(a.data, b.data)

    def test_shift_semantics_against_reimplementation(self, tk, rng):
        s = sino2d(rng)
        out = host(tk.add_detector_jitter(s, 2, "u", seed=7))
        shifts = tk.artifacts.jitter_shifts(7, s.n_projections, 2)
        assert set(shifts.tolist()) <= {-2, -1, 0, 1, 2} and len(set(shifts.tolist())) > 1
        src = host(s)
        for i, shift in enumerate(shifts):
            row = src[i]
            expect = np.zeros_like(row)
            if shift > 0:
                expect[shift:] = row[:-shift]
            elif shift < 0:
                expect[:shift] = row[-shift:]
            else:
                expect = row
            np.testing.assert_array_equal(out[i], expect)

    def test_v_axis(self, tk, rng):
        s = sino3d(rng)
        out = host(tk.add_detector_jitter(s, 1, "v", seed=3))
        shifts = tk.artifacts.jitter_shifts(3, s.n_projections, 1)
        src = host(s)
        for i, sh in enumerate(shifts):
            np.testing.assert_array_equal(out[i], np.roll(src[i], sh, axis=0) * (
                (np.arange(src.shape[1]) - sh >= 0) & (np.arange(src.shape[1]) - sh < src.shape[1]))[:, None])

    def test_offsets_uniform(self, tk):
        sh = tk.artifacts.jitter_shifts(11, 20000, 3)
        counts = np.bincount(sh + 3, minlength=7)
        assert abs(sh.mean()) < 0.05 and counts.min() > 2500  # 7 values x ~2857

    def test_invalid(self, tk, rng):
        with pytest.raises(ValueError):
            tk.add_detector_jitter(sino2d(rng), 1, "v", seed=0)
        with pytest.raises(ValueError):
            tk.add_detector_jitter(sino2d(rng), -1, "u", seed=0)


@pytest.mark.gpu
class TestPoissonNoise:
    def test_zero_line_integral_unbiased(self, tk):
        i0, n = 1e4, 10_000
        out = tk.add_poisson_noise(tk.Sinogram(np.zeros((100, 100)), (1.0,)), i0, "transmission", seed=123)
        assert abs(host(out).mean()) < 3 * (1.0 / np.sqrt(i0)) / np.sqrt(n)

    def test_attenuated_value_recovered(self, tk):
        out = tk.add_poisson_noise(tk.Sinogram(np.full((100, 100), 2.0), (1.0,)), 1e6, "transmission", seed=99)
        assert abs(host(out).mean() - 2.0) < 0.01

    def test_transmission_variance_matches_delta_method(self, tk):
        # Var(-ln(N / i0)) ~ 1 / (i0 e^-p) for large counts
        p, i0 = 1.0, 1e4
        out = host(tk.add_poisson_noise(tk.Sinogram(np.full((200, 300), p), (1.0,)), i0, "transmission", seed=4))
        assert out.var() == pytest.approx(1.0 / (i0 * np.exp(-p)), rel=0.03)

    @pytest.mark.parametrize("lam", [0.3, 7.0, 55.0, 3000.0])
    def test_direct_mode_mean_and_variance(self, tk, lam):
        out = host(tk.add_poisson_noise(tk.Sinogram(np.full((200, 250), lam), (1.0,)), 1.0, "direct", seed=17))
        n = out.size
        assert out.mean() == pytest.approx(lam, abs=4 * np.sqrt(lam / n))
        assert out.var() == pytest.approx(lam, rel=0.05)
        assert (out == np.round(out)).all()

    def test_same_seed_identical_and_seeds_differ(self, tk, rng):
        s = sino2d(rng)
        a = tk.add_poisson_noise(s, 1e5, "transmission", seed=5)
        b = tk.add_poisson_noise(s, 1e5, "transmission", seed=5)
        c = tk.add_poisson_noise(s, 1e5, "transmission", seed=6)
        assert torch.equal(a.data, b.data) and not torch.equal(a.data, c.data)

    def test_transmission_mad_decreases_with_dose(self, tk, rng):
        s = sino2d(rng, n=32, w=64)
        mads = [np.mean(np.abs(host(tk.add_poisson_noise(s, i0, "transmission", seed=1)) - host(s)))
                for i0 in (1e3, 1e5)]
        assert mads[1] < mads[0]

    def test_invalid_inputs_rejected(self, tk, rng):
        with pytest.raises(ValueError):
            tk.add_poisson_noise(sino2d(rng), 0.0, "transmission", seed=0)
        with pytest.raises(ValueError):
            tk.add_poisson_noise(tk.Sinogram(np.array([[-0.5, 1.0]]), (1.0,)), 1e4, "transmission", seed=0)
        with pytest.raises(ValueError):
            tk.add_poisson_noise(sino2d(rng), 1e4, "bogus", seed=0)


@pytest.mark.gpu
class TestGaussianNoise:
    def test_zero_std_adds_mean_exactly(self, tk, rng):
        s = sino2d(rng)
        out = tk.add_gaussian_noise(s, mean=0.25, std=0.0, seed=8)
        np.testing.assert_array_equal(host(out), (host(s) + 0.25).astype(np.float32))

    def test_sample_statistics(self, tk):
        s = tk.Sinogram(np.zeros((400, 300)), (1.0,))
        mean, std = 0.4, 1.3
        d = host(tk.add_gaussian_noise(s, mean, std, seed=21))
        assert abs(d.mean() - mean) < 0.01 * max(1.0, abs(mean)) + 3 * std / np.sqrt(d.size)
        assert abs(d.std() - std) < 0.01 * std

    def test_per_view_streams_independent(self, tk):
        d = host(tk.add_gaussian_noise(tk.Sinogram(np.zeros((2, 50000)), (1.0,)), 0.0, 1.0, seed=2))
        assert abs(np.corrcoef(d[0], d[1])[0, 1]) < 0.02

    def test_negative_std_rejected(self, tk, rng):
        with pytest.raises(ValueError):
            tk.add_gaussian_noise(sino2d(rng), 0.0, -1.0, seed=0)


@pytest.mark.gpu
class TestRingAndBlur:
    def test_zero_mode_clears_only_the_selection(self, tk, rng):
        s = sino2d(rng, n=20, w=30)
        out = host(tk.add_ring_artifact(s, columns=[4, 17], projection_range=(5, 12), mode="zero"))
        assert (out[5:12][:, [4, 17]] == 0).all()
        mask = np.ones(out.shape, dtype=bool)
        mask[5:12, 4] = mask[5:12, 17] = False
        np.testing.assert_array_equal(out[mask], host(s)[mask])

    def test_identities(self, tk, rng):
        s = sino2d(rng)
        assert torch.equal(tk.add_ring_artifact(s, [3], (0, s.n_projections), mode="scale", factor=1.0).data,
                           s.data)
        assert torch.equal(tk.add_ring_artifact(s, [3], (7, 7), mode="zero").data, s.data)
        geom = tk.circular_cone_geometry((16, 16, 16), (1, 1, 1), (20, 24), (1.0, 1.0), 8, 2 * np.pi,
                                         1200.0, 750.0)
        s3 = sino3d(rng, n=8)
        assert torch.equal(tk.add_gantry_motion_blur(s3, geom, 1).data, s3.data)

    def test_impulse_spreads_along_u_at_theta_zero(self, tk):
        geom = tk.circular_cone_geometry((16, 16, 16), (1, 1, 1), (20, 24), (1.0, 1.0), 4, 2 * np.pi,
                                         1200.0, 750.0)
        img = np.zeros((4, 20, 24))
        img[0, 10, 12] = 1.0
        out = host(tk.add_gantry_motion_blur(tk.Sinogram(img, (1.0, 1.0)), geom, 5))
        np.testing.assert_allclose(out[0, 10, 10:15], 0.2, atol=1e-7)
        assert out[0].sum() == pytest.approx(1.0, abs=1e-6)
        assert (np.delete(out[0, 10], np.s_[10:15]) == 0).all()

    def test_invalid(self, tk, rng):
        s = sino2d(rng, w=30)
        with pytest.raises(ValueError):
            tk.add_ring_artifact(s, [30], (0, 5), mode="zero")
        with pytest.raises(ValueError):
            tk.add_ring_artifact(s, [3], (0, 99), mode="zero")
        with pytest.raises(ValueError):
            tk.add_ring_artifact(s, [3], (0, 5), mode="scale")
        geom = tk.circular_cone_geometry((16, 16, 16), (1, 1, 1), (20, 24), (1.0, 1.0), 8, 2 * np.pi,
                                         1200.0, 750.0)
        with pytest.raises(ValueError):
            tk.add_gantry_motion_blur(sino3d(rng, n=8), geom, 4)

    def test_full_size_throughput_smoke(self, tk):
        """cfg4-sized sinogram (720 x 1024^2): each simulator runs on the device and keeps shape."""
        s = tk.Sinogram(torch.rand(720, 1024, 1024, device="cuda") * 3, (0.6, 0.6))
        geom = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * np.pi,
                                         1200.0, 750.0)
        for out in (tk.add_poisson_noise(s, 1e5, seed=1), tk.add_gaussian_noise(s, 0.0, 0.01, seed=1),
                    tk.add_detector_jitter(s, 2, "u", seed=1), tk.add_ring_artifact(s, [100, 500], None, "zero"),
                    tk.add_gantry_motion_blur(s, geom, 5)):
            assert out.data.shape == s.data.shape and bool(torch.isfinite(out.data).all())


@pytest.mark.gpu
def test_config_artifact_chain(tk, rng):
    """PipelineConfig.apply_artifacts runs the reference's chain schema (config.py:208-258)."""
    from paper_2511_08427_b200.config import ConfigError, PipelineConfig

    base = {"geometry_kind": "cone3d", "volume_shape": [16, 16, 16], "volume_spacing": [1, 1, 1],
            "detector_shape": [20, 24], "detector_spacing": [1.0, 1.0], "number_of_projections": 6,
            "angular_range": 2 * np.pi, "sdd": 1200.0, "sid": 750.0}
    chain = [{"kind": "poisson", "i0": 1e5, "seed": 3}, {"kind": "ring", "columns": [2], "mode": "zero"},
             {"kind": "gantry_blur", "kernel_len_px": 3}, {"kind": "gaussian", "std": 0.0, "mean": 0.5}]
    cfg = PipelineConfig.from_dict({**base, "artifacts": chain})
    geom = cfg.build_geometry()
    s = sino3d(rng)
    out = cfg.apply_artifacts(s, geom)
    want = tk.add_gaussian_noise(tk.add_gantry_motion_blur(tk.add_ring_artifact(
        tk.add_poisson_noise(s, 1e5, seed=3), [2]), geom, 3), 0.5, 0.0)
    assert torch.equal(out.data, want.data)
    for bad in ([{"kind": "nope"}], [{"kind": "poisson"}], [{"kind": "gaussian", "std": 1.0, "extra": 1}],
                [{"kind": "poisson", "i0": -1.0}]):
        with pytest.raises(ConfigError):
            PipelineConfig.from_dict({**base, "artifacts": bad}).apply_artifacts(s, geom)
