"""CPU-only tests: the C ABI library loads and exports the header's symbols, and
the host-side logic (geometry, config, filter weights, boundary validation)
matches the reference's golden vectors.  No kernel is launched here."""

import json
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2511_08427_b200 as tk
from paper_2511_08427_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


class TestAbi:
    def test_library_exports_every_header_symbol(self):
        header = (ROOT / "include" / "tk_b200.h").read_text()
        names = set(re.findall(r"\b(tk_[a-z0-9_]+)\s*\(", header))
        assert len(names) >= 18
        lib = _lib.load()
        missing = [n for n in sorted(names) if not hasattr(lib, n)]
        assert not missing, missing
        assert names <= set(_lib.SIGNATURES), sorted(names - set(_lib.SIGNATURES))

    def test_version_and_errors_without_device_work(self):
        lib = _lib.load()
        assert _lib.version() >= 10000
        # argument validation runs before any CUDA call
        rc = lib.tk_forward_cone_3d(None, 1, 1, 1, 1.0, 1.0, 1.0, None, None, 1, 1, 1, 0.5, None, None)
        assert rc == 1 and b"null pointer" in lib.tk_last_error()

    def test_built_for_sm100a(self):
        import subprocess

        out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
        if out.returncode != 0:
            pytest.skip("cuobjdump unavailable")
        assert "sm_100a" in out.stdout


class TestGeometryGolden:
    def test_circular_matrices(self, golden):
        g = golden("geometry")
        geom = tk.circular_cone_geometry((16, 16, 16), (1, 1, 1), (12, 12), (1.6, 1.6), 8, 2 * np.pi, 1200.0, 750.0)
        np.testing.assert_allclose(geom.matrix_array(), g["mats"], rtol=0, atol=1e-9)
        src, minv = geom.ray_constants
        np.testing.assert_allclose(src, g["sources"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(minv, g["minv"], rtol=1e-12, atol=1e-15)
        g4 = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * np.pi, 1200.0, 750.0)
        np.testing.assert_allclose(g4.matrix_array(), g["mats4"], rtol=0, atol=1e-7)

    def test_pose_trajectories(self, golden):
        g = golden("geometry")
        th = np.linspace(0, 4 * np.pi, 10, endpoint=False)
        poses = []
        for t in th:
            zc = -6.0 + 12.0 * t / (4 * np.pi)
            c, s = np.cos(t), np.sin(t)
            poses.append(tk.Pose([750 * c, 750 * s, zc], [-450 * c, -450 * s, zc], [-s, c, 0], [0, 0, 1]))
        m = np.stack([p.entries for p in tk.trajectory_from_poses(poses, (10, 14), (1.5, 1.8))])
        np.testing.assert_allclose(m, g["mats_helix"], rtol=0, atol=1e-9)
        hel = tk.helical_trajectory_3d(10, 4 * np.pi, 1200.0, 750.0, (10, 14), (1.5, 1.8), -6.0, 6.0)
        np.testing.assert_allclose(np.stack([p.entries for p in hel]), g["mats_helix"], rtol=0, atol=1e-9)
        sin = tk.sinusoidal_trajectory_3d(9, 2 * np.pi, 1200.0, 750.0, (12, 12), (1.6, 1.6), 4.0, 2.0)
        np.testing.assert_allclose(np.stack([p.entries for p in sin]), g["mats_sin"], rtol=0, atol=1e-9)

    def test_from_raw_and_json_roundtrip(self, golden, tmp_path):
        g = golden("geometry")
        np.testing.assert_allclose(tk.ProjectionMatrix.from_raw(g["raw"]).entries, g["from_raw"], atol=1e-12)
        mats = tk.circular_trajectory_3d(5, 2 * np.pi, 1200.0, 750.0, (12, 12), (1.6, 1.6))
        tk.save_projection_matrices(mats, tmp_path / "m.json")
        back = tk.load_projection_matrices(tmp_path / "m.json")
        for a, b in zip(mats, back):  # reload renormalises the third row (from_raw)
            np.testing.assert_allclose(a.entries, b.entries, rtol=1e-14, atol=1e-9)

    def test_validation(self):
        with pytest.raises(ValueError):
            tk.Pose([0, 0, 0], [1, 0, 0], [0, 1.1, 0], [0, 0, 1])
        with pytest.raises(tk.DegeneratePoseError):
            tk.trajectory_from_poses([tk.Pose([0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]),
                                      tk.Pose([0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1])], (4, 4), (0, 1))
        with pytest.raises(ValueError):
            tk.GeometryFan2D((8, 8), (1, 1), 8, 1.0, [0.0], sdd=500.0, sid=750.0)
        with pytest.raises(ValueError, match="rank 3"):
            tk.ProjectionMatrix(np.zeros((3, 4)))

    def test_pyronn_geometry_front_end(self):
        g = tk.Geometry().init_from_parameters([16, 16, 16], [1, 1, 1], [12, 12], [1.6, 1.6], 8, 2 * np.pi,
                                               source_isocenter_distance=750.0,
                                               source_detector_distance=1200.0).build()
        ref = tk.circular_cone_geometry((16, 16, 16), (1, 1, 1), (12, 12), (1.6, 1.6), 8, 2 * np.pi, 1200.0, 750.0)
        np.testing.assert_array_equal(g.matrix_array(), ref.matrix_array())
        params = dict(volume_shape=[16, 16, 16], volume_spacing=[1, 1, 1], detector_shape=[12, 12],
                      detector_spacing=[1.6, 1.6], number_of_projections=8, angular_range=2 * np.pi,
                      sdd=1200, sid=750)
        g2 = tk.GeometryCone3D(**params)
        g2.set_trajectory(tk.circular_trajectory_3d(**params))
        np.testing.assert_array_equal(g2.matrix_array(), ref.matrix_array())


class TestFilterWeights:
    @pytest.mark.parametrize("kind,make", [("ramp", tk.ramp_filter), ("shepp_logan", tk.shepp_logan_filter),
                                           ("cosine", tk.cosine_filter)])
    @pytest.mark.parametrize("width,sp", [(12, 1.0), (48, 0.625), (100, 1.3), (1024, 0.375)])
    def test_weights_match_reference(self, golden, kind, make, width, sp):
        w = make(width, sp).weights
        np.testing.assert_allclose(w, golden("filters")[f"{kind}_{width}"], rtol=1e-13, atol=1e-13 * sp ** -2)
        assert (w[1:] == w[:0:-1]).all()  # bit-exact symmetry (reference test_filters.py:45-47)

    def test_padding_and_pitch(self):
        assert tk.ramp_filter(100, 1.0).n_pad == 256
        assert tk.ramp_filter(128, 1.0).n_pad == 256
        assert tk.ramp_filter(129, 1.0).n_pad == 512
        gf = tk.GeometryFan2D((32, 32), (1, 1), 48, 1.0, tk.circular_trajectory_2d(12, 2 * np.pi), sdd=1200, sid=750)
        assert tk.reconstruction_filter(gf, "ramp").detector_spacing == pytest.approx(750 / 1200)
        with pytest.raises(ValueError):
            tk.reconstruction_filter(gf, "hann")

    def test_pyronn_filter_builders(self):
        params = dict(detector_shape=[400, 600], detector_spacing=[1, 1], sdd=1200, sid=750)
        f = tk.shepp_logan_3D(**params)
        ref = tk.shepp_logan_filter(600, 750 / 1200)
        np.testing.assert_array_equal(f.weights, ref.weights)


class TestConfig:
    CONE = {"geometry_kind": "cone3d", "volume_shape": [16, 16, 16], "volume_spacing": [1.0, 1.0, 1.0],
            "detector_shape": [12, 12], "detector_spacing": [1.6, 1.6], "number_of_projections": 8,
            "angular_range": 2 * np.pi, "sdd": 1200.0, "sid": 750.0}

    def test_build_and_memoise(self, golden):
        cfg = tk.PipelineConfig.from_dict(self.CONE)
        g1 = cfg.build_geometry()
        assert cfg.build_geometry() is g1
        np.testing.assert_allclose(g1.matrix_array(), golden("geometry")["mats"], atol=1e-9)

    def test_errors_name_the_field(self):
        bad = dict(self.CONE)
        del bad["sdd"]
        with pytest.raises(tk.ConfigError, match="sdd"):
            tk.PipelineConfig.from_dict(bad)
        with pytest.raises(tk.ConfigError, match="geometry_kind"):
            tk.PipelineConfig.from_dict({"geometry_kind": "nope"})
        with pytest.raises(tk.ConfigError, match="step_scale"):
            tk.PipelineConfig.from_dict(dict(self.CONE, step_scale=0.0))

    def test_matrices_path(self, tmp_path):
        mats = tk.helical_trajectory_3d(8, 2 * np.pi, 1200.0, 750.0, (12, 12), (1.6, 1.6), -5.0, 5.0)
        tk.save_projection_matrices(mats, tmp_path / "traj.json")
        doc = dict(self.CONE, matrices_path="traj.json")
        (tmp_path / "c.json").write_text(json.dumps(doc))
        g = tk.load_config(tmp_path / "c.json").build_geometry()
        np.testing.assert_allclose(g.matrix_array(), np.stack([m.entries for m in mats]), atol=1e-12)


class TestBoundaryValidation:
    CFG = {"geometry_kind": "parallel2d", "volume_shape": [32, 32], "volume_spacing": [1.0, 1.0],
           "detector_shape": [48], "detector_spacing": [1.0], "number_of_projections": 24,
           "angular_range": 2 * np.pi}

    def test_shape_dtype_layout(self):
        from paper_2511_08427_b200 import ops

        with pytest.raises(ops.BoundaryError) as err:
            ops.py_forward_project(np.zeros((16, 16), np.float32), self.CFG)
        assert "(32, 32)" in str(err.value) and "(16, 16)" in str(err.value)
        with pytest.raises(ops.BoundaryError, match="contiguous"):
            ops.py_forward_project(np.zeros((32, 64), np.float32)[:, ::2], self.CFG)
        with pytest.raises(ops.BoundaryError, match="float32"):
            ops.py_forward_project(np.zeros((32, 32)), self.CFG)
        with pytest.raises(Exception):
            ops.py_forward_project(np.zeros((32, 32), np.float32), {"geometry_kind": "nope"})

    def test_no_cpu_fallback(self):
        import torch

        if torch.cuda.is_available():
            pytest.skip("has a GPU")
        from paper_2511_08427_b200 import ops

        with pytest.raises(RuntimeError, match="CUDA"):
            ops.py_forward_project(np.zeros((32, 32), np.float32), self.CFG)


class TestRowBands:
    def test_band_covers_every_voxel_projection(self):
        from paper_2511_08427_b200 import distributed as D

        geom = tk.circular_cone_geometry((64, 48, 40), (0.5, 0.6, 0.7), (80, 90), (0.6, 0.6), 36, 2 * np.pi, 1200.0, 750.0)
        nz, ny, nx = geom.volume_shape
        sz, sy, sx = geom.volume_spacing
        mats = geom.matrix_array()
        for world in (2, 4, 8):
            for rank in range(world):
                z0, z1 = D.shard_bounds(nz, world, rank)
                r0, r1 = D.row_band(geom, z0, z1)
                z = (np.arange(z0, z1) - (nz - 1) / 2) * sz
                y = (np.arange(ny) - (ny - 1) / 2) * sy
                x = (np.arange(nx) - (nx - 1) / 2) * sx
                Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
                pts = np.stack([X.ravel(), Y.ravel(), Z.ravel(), np.ones(X.size)])
                hom = mats @ pts
                fr = hom[:, 1] / hom[:, 2]
                lo = np.floor(fr.min())
                hi = np.floor(fr.max()) + 1
                assert r0 <= max(lo, 0) and r1 - 1 >= min(hi, geom.detector_shape[0] - 1)

    def test_shard_bounds_partition(self):
        from paper_2511_08427_b200 import distributed as D

        for n, w in ((720, 8), (512, 3), (5, 8)):
            spans = [D.shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_tapered_pipeline_chunks_cover_views_once():
    """ops._tapered: the copy/compute pipelines' view chunks partition [0, n) in
    order, with the short chunk at the head (H2D pipelines) or tail (D2H)."""
    from paper_2511_08427_b200.ops import _tapered

    for n in (1, 2, 5, 37, 720, 1001):
        for parts in (1, 3, 12):
            for small in (0, 1, 8, 12):
                for head in (True, False):
                    for align in (1, 8):
                        ch = _tapered(n, parts, small, head, align)
                        assert ch[0][0] == 0 and ch[-1][1] == n
                        assert all(b < e for b, e in ch)
                        assert all(ch[i][1] == ch[i + 1][0] for i in range(len(ch) - 1))
                        want = -(-max(1, small) // align) * align
                        if n > want:
                            short = ch[0] if head else ch[-1]
                            assert short[1] - short[0] == want
                            # every other chunk but the one before the short tail is aligned
                            body = ch[1:] if head else ch[:-1]
                            assert all((e - b) % align == 0 for b, e in body[:-1])


def test_bp_tile_bank_model_supports_the_8x4_warp_and_pitch_rule():
    """The back projector's warp footprint / tile pitch choice (tk_bp_tma.cu) rests on
    scripts/bp_bank_model.py: at cfg4, 8 x 4 warps with a pitch == 12 or 20 (mod 32)
    need ~1 LDS wavefront per instruction, 16 x 2 warps ~1.3."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bp_bank_model", ROOT / "scripts" / "bp_bank_model.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    views = range(30, 720, 90)  # oblique and near-axis views
    blocks = ((3, 5, 2), (16, 16, 8), (28, 9, 13))
    assert m.model(52, 8, 4, views, blocks) < 1.05
    assert m.model(44, 8, 4, views, blocks) < 1.05
    assert m.model(52, 16, 2, views, blocks) > 1.25


class TestForwardKernelChoice:
    """tk_forward_cone_3d_path: the z-mirror-pair kernel runs exactly for
    z-mirror-symmetric scans whose volume fits its layout (host-only query)."""

    def test_circular_orbits_use_the_mirror_kernel(self, monkeypatch):
        from paper_2511_08427_b200.projectors import forward_kernel_path

        monkeypatch.setenv("TK_FP_MIRROR", "1")
        for shape, det in [((512,) * 3, (1024, 1024)), ((256,) * 3, (512, 512)), ((33, 40, 21), (31, 45)),
                           ((16, 16, 16), (12, 12))]:
            g = tk.circular_cone_geometry(shape, (0.5,) * 3, det, (0.6, 0.6), 36, 2 * np.pi, 1200.0, 750.0)
            assert forward_kernel_path(g) == "mirror", (shape, det)

    def test_other_scans_use_the_general_kernel(self, monkeypatch):
        from paper_2511_08427_b200.projectors import forward_kernel_path

        monkeypatch.setenv("TK_FP_MIRROR", "1")
        det, ds = (64, 64), (1.6, 1.6)
        helix = tk.helical_trajectory_3d(36, 4 * np.pi, 1200.0, 750.0, det, ds, -20.0, 20.0)
        g = tk.GeometryCone3D((32,) * 3, (1,) * 3, det, ds, helix, 1200.0, 750.0)
        assert forward_kernel_path(g) == "general"
        sinus = tk.sinusoidal_trajectory_3d(36, 2 * np.pi, 1200.0, 750.0, det, ds, 20.0)
        g = tk.GeometryCone3D((32,) * 3, (1,) * 3, det, ds, sinus, 1200.0, 750.0)
        assert forward_kernel_path(g) == "general"
        # detector shifted by a fraction of a row: rays no longer pair up
        circ = tk.circular_cone_geometry((32,) * 3, (1,) * 3, det, ds, 36, 2 * np.pi, 1200.0, 750.0)
        mats = circ.matrix_array().copy()
        mats[:, 1, :] += 0.3 * mats[:, 2, :]
        g = tk.GeometryCone3D((32,) * 3, (1,) * 3, det, ds, [tk.ProjectionMatrix(m) for m in mats], 1200.0, 750.0)
        assert forward_kernel_path(g) == "general"
        # too large for 32-bit cell indices of the pair layout
        g = tk.circular_cone_geometry((2048,) * 3, (0.125,) * 3, det, ds, 4, 2 * np.pi, 1200.0, 750.0)
        assert forward_kernel_path(g) == "general"
        monkeypatch.setenv("TK_FP_MIRROR", "0")
        assert forward_kernel_path(circ) == "general"
