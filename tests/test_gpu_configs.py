"""GPU parity at the BASELINE.json configurations, at full size.

Every case compares the CUDA path (through libtkb200.so) with the float64 C
oracle (`oracle/tk_oracle.c`, bit-exact to the reference kernels on the golden
fixtures) on identical inputs.  Tolerance: the north star's relative L2 <= 1e-4
on sinograms and volumes; dot tests: <A x, y> vs <x, A^T y> <= 1e-4 relative for
the matched transposes, and the reference's own bound (1e-2,
/root/reference/pkg/tests/test_projectors.py:246-277) for the paired (unmatched)
A/B, whose defect must also agree with the oracle's own defect on the same
inputs.

Inputs are the survey's: Shepp-Logan phantoms and uniform[0,1) / N(0,1) arrays
from numpy's default_rng(20240917) (the reference suite's seed,
pkg/tests/conftest.py:18-20).
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-4
SDD, SID = 1200.0, 750.0
SEED = 20240917


def rel(got, want):
    got = np.asarray(got.detach().cpu().numpy() if isinstance(got, torch.Tensor) else got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


def f32(a):
    """The float32 array both sides see (the GPU takes float32; the oracle gets
    the same values widened to float64)."""
    return np.asarray(a, np.float32).astype(np.float64)


@pytest.fixture(scope="module")
def tk(cuda):
    import paper_2511_08427_b200 as tk

    return tk


def paired_defect(Ax, y, x, By):
    """The reference's adjoint-pairing defect (test_projectors.py:247-250)."""
    Ax, y, x, By = (np.asarray(a, np.float64).ravel() for a in (Ax, y, x, By))
    return abs(Ax @ y - x @ By) / (np.linalg.norm(Ax) * np.linalg.norm(y))


# ---------------------------------------------------------------------------
# cfg1: parallel 256^2 @1 mm, 180 angles over pi, 367 px @1 mm: FP + FBP
# ---------------------------------------------------------------------------


class TestCfg1Parallel:
    @pytest.fixture(scope="class")
    def setup(self, tk):
        ang = tk.circular_trajectory_2d(180, np.pi)
        geom = tk.GeometryParallel2D((256, 256), (1.0, 1.0), 367, 1.0, ang)
        x = f32(tk.phantoms.shepp_logan_2d((256, 256)).cpu().numpy())
        return geom, ang, x

    def test_forward(self, tk, oracle, setup):
        geom, ang, x = setup
        got = tk.forward_project(tk.Volume(x, (1, 1)), geom).data
        assert rel(got, oracle.forward_parallel_2d(x, (1, 1), ang, 367, 1.0, 0.5)) < TOL

    @pytest.mark.parametrize("kind", ["ramp", "shepp_logan", "cosine"])
    def test_fbp(self, tk, oracle, setup, kind):
        geom, ang, x = setup
        sino = f32(oracle.forward_parallel_2d(x, (1, 1), ang, 367, 1.0, 0.5))
        got = tk.fbp_parallel_2d(tk.Sinogram(sino, (1.0,)), geom, kind).data
        want = oracle.fbp_parallel_2d(sino, ang, 1.0, (256, 256), (1, 1), kind)
        assert rel(got, want) < TOL

    def test_fp_then_fbp_chain(self, tk, oracle, setup):
        """The whole GPU chain (FP -> filter -> BP -> pi/V) against the oracle's chain."""
        geom, ang, x = setup
        sino = tk.forward_project(tk.Volume(x, (1, 1)), geom)
        got = tk.fbp_parallel_2d(sino, geom, "shepp_logan").data
        want = oracle.fbp_parallel_2d(oracle.forward_parallel_2d(x, (1, 1), ang, 367, 1.0, 0.5), ang, 1.0,
                                      (256, 256), (1, 1), "shepp_logan")
        assert rel(got, want) < TOL


# ---------------------------------------------------------------------------
# cfg2: fan 512^2 @1 mm, 360 angles over 2 pi, 768 px @1.6 mm: FP + BP + adjoint test
# ---------------------------------------------------------------------------


class TestCfg2Fan:
    @pytest.fixture(scope="class")
    def setup(self, tk):
        ang = tk.circular_trajectory_2d(360, 2 * np.pi)
        geom = tk.GeometryFan2D((512, 512), (1.0, 1.0), 768, 1.6, ang, sdd=SDD, sid=SID)
        return geom, ang

    def test_forward_shepp_logan(self, tk, oracle, setup):
        geom, ang = setup
        x = f32(tk.phantoms.shepp_logan_2d((512, 512)).cpu().numpy())
        got = tk.forward_project(tk.Volume(x, (1, 1)), geom).data
        assert rel(got, oracle.forward_fan_2d(x, (1, 1), ang, SDD, SID, 768, 1.6, 0.5)) < TOL

    @pytest.mark.parametrize("weighted", [False, True])
    def test_back(self, tk, oracle, setup, weighted):
        geom, ang = setup
        y = f32(np.random.default_rng(SEED).standard_normal((360, 768)))
        got = tk.back_project(tk.Sinogram(y, (1.6,)), geom, fdk_weighting=weighted).data
        want = oracle.back_fan_2d(y, ang, SDD, SID, 1.6, (512, 512), (1, 1), weighted)
        assert rel(got, want) < TOL

    @pytest.mark.parametrize("kind", ["ramp", "shepp_logan"])
    def test_fbp(self, tk, oracle, setup, kind):
        geom, ang = setup
        x = f32(tk.phantoms.shepp_logan_2d((512, 512)).cpu().numpy())
        sino = f32(oracle.forward_fan_2d(x, (1, 1), ang, SDD, SID, 768, 1.6, 0.5))
        got = tk.fbp_fan_2d(tk.Sinogram(sino, (1.6,)), geom, kind).data
        want = oracle.fbp_fan_2d(sino, ang, SDD, SID, 1.6, (512, 512), (1, 1), kind)
        assert rel(got, want) < TOL

    def test_adjoint_paired_and_matched(self, tk, oracle, setup):
        """The config's defining check on N(0,1) inputs.

        * paired (reference) A/B: defect below the reference's bound (1e-2) and
          equal to the oracle's own defect on the same x, y (the GPU pair IS the
          reference pair, so the two defects agree to fp32 accuracy);
        * matched A^T: <A x, y> vs <x, A^T y> <= 1e-4 relative (north star).
        """
        from paper_2511_08427_b200.projectors import fp_adjoint_tensor, fp_tensor

        geom, ang = setup
        rng = np.random.default_rng(SEED)
        for _ in range(3):
            x = f32(rng.standard_normal((512, 512)))
            y = f32(rng.standard_normal((360, 768)))
            Ax = tk.forward_project(tk.Volume(x, (1, 1)), geom).data.cpu().numpy()
            By = tk.back_project(tk.Sinogram(y, (1.6,)), geom).data.cpu().numpy()
            d_gpu = paired_defect(Ax, y, x, By)
            Ax_o = oracle.forward_fan_2d(x, (1, 1), ang, SDD, SID, 768, 1.6, 0.5)
            By_o = oracle.back_fan_2d(y, ang, SDD, SID, 1.6, (512, 512), (1, 1), False)
            d_ora = paired_defect(Ax_o, y, x, By_o)
            assert d_gpu < 1e-2
            assert abs(d_gpu - d_ora) < 1e-5 + 1e-3 * d_ora, (d_gpu, d_ora)
            xt = torch.as_tensor(x, dtype=torch.float32, device="cuda")
            yt = torch.as_tensor(y, dtype=torch.float32, device="cuda")
            lhs = float((fp_tensor(xt, geom, 0.5).double() * yt.double()).sum())
            rhs = float((xt.double() * fp_adjoint_tensor(yt, geom, 0.5).double()).sum())
            assert abs(lhs - rhs) / max(abs(lhs), abs(rhs)) < TOL, (lhs, rhs)


# ---------------------------------------------------------------------------
# cfg3: cone 256^3 @1 mm, 360 views over 2 pi, 512^2 @1.2 mm: FDK (full size)
# ---------------------------------------------------------------------------


class TestCfg3Cone:
    @pytest.fixture(scope="class")
    def setup(self, tk, oracle):
        geom = tk.circular_cone_geometry((256,) * 3, (1.0,) * 3, (512, 512), (1.2, 1.2), 360, 2 * np.pi,
                                         SDD, SID)
        x = f32(oracle.shepp_logan_3d((256,) * 3))
        mats = geom.matrix_array()
        sino = oracle.forward_cone_3d(x, (1, 1, 1), mats, (512, 512), 0.5)  # all 360 views
        return geom, mats, x, sino

    def test_forward_all_views(self, tk, setup):
        geom, mats, x, sino = setup
        got = tk.forward_project(tk.Volume(x, (1, 1, 1)), geom).data
        assert rel(got, sino) < TOL

    def test_fdk_from_oracle_sinogram(self, tk, oracle, setup):
        geom, mats, x, sino = setup
        s32 = f32(sino)
        want = oracle.fdk_cone_3d(s32, mats, SDD, SID, (1.2, 1.2), (256,) * 3, (1, 1, 1), "shepp_logan")
        got = tk.fdk_cone_3d(tk.Sinogram(s32, (1.2, 1.2)), geom, "shepp_logan").data
        assert rel(got, want) < TOL

    def test_fdk_gpu_chain(self, tk, oracle, setup):
        """GPU FP -> GPU filter -> GPU weighted BP -> pi/V against the oracle's chain."""
        geom, mats, x, sino = setup
        want = oracle.fdk_cone_3d(sino, mats, SDD, SID, (1.2, 1.2), (256,) * 3, (1, 1, 1), "shepp_logan")
        y = tk.forward_project(tk.Volume(x, (1, 1, 1)), geom)
        got = tk.fdk_cone_3d(y, geom, "shepp_logan").data
        assert rel(got, want) < TOL


# ---------------------------------------------------------------------------
# cfg4: 512^3 @0.5 mm, 1024^2 @0.6 mm, 720 views -- a view subset of the orbit
# at full resolution, on the survey's uniform[0,1) phantom, through the GPU
# FP -> filter -> BP chain the bench times
# ---------------------------------------------------------------------------


class TestCfg4Subset:
    VIEWS = [0, 45, 90, 200, 270, 405, 555, 630]  # axis-aligned and oblique

    @pytest.fixture(scope="class")
    def setup(self, tk):
        full = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * np.pi,
                                         SDD, SID)
        mats = full.matrix_array()[self.VIEWS]
        geom = tk.GeometryCone3D((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6),
                                 [tk.ProjectionMatrix(m) for m in mats], SDD, SID)
        x = np.random.default_rng(SEED).random((512,) * 3, dtype=np.float32).astype(np.float64)
        return geom, mats, x

    def test_uniform_fp_and_fdk_chain(self, tk, oracle, setup):
        geom, mats, x = setup
        want_fp = oracle.forward_cone_3d(x, (0.5,) * 3, mats, (1024, 1024), 0.25)
        xt = torch.as_tensor(x, dtype=torch.float32, device="cuda")
        fp = tk.forward_project(tk.Volume(xt, (0.5,) * 3), geom)
        assert rel(fp.data, want_fp) < TOL
        # the bench's FDK: GPU filter -> GPU weighted BP (TMA) -> pi/V, on the GPU sinogram,
        # against the oracle's FDK of the oracle sinogram
        got = tk.fdk_cone_3d(fp, geom, "shepp_logan").data
        want = oracle.fdk_cone_3d(want_fp, mats, SDD, SID, (0.6, 0.6), (512,) * 3, (0.5,) * 3, "shepp_logan")
        assert rel(got, want) < TOL
        # the filter alone on the same (float32) input
        s32 = f32(want_fp)
        got_f = tk.filter_stage(tk.Sinogram(s32, (0.6, 0.6)), geom, "shepp_logan").data
        want_f = oracle.filter_stage_cone(s32, SDD, SID, (0.6, 0.6), "shepp_logan")
        assert rel(got_f, want_f) < TOL

    def test_shepp_logan_fdk_chain(self, tk, oracle, setup):
        geom, mats, _ = setup
        x = f32(oracle.shepp_logan_3d((512,) * 3))
        want_fp = oracle.forward_cone_3d(x, (0.5,) * 3, mats, (1024, 1024), 0.25)
        fp = tk.forward_project(tk.Volume(x, (0.5,) * 3), geom)
        assert rel(fp.data, want_fp) < TOL
        got = tk.fdk_cone_3d(fp, geom, "shepp_logan").data
        want = oracle.fdk_cone_3d(want_fp, mats, SDD, SID, (0.6, 0.6), (512,) * 3, (0.5,) * 3, "shepp_logan")
        assert rel(got, want) < TOL
