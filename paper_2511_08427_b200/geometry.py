"""Acquisition geometry: beam geometries, trajectories and 3x4 projection matrices.

Host-side (float64, numpy) mirror of the reference geometry module
(/root/reference/pkg/src/tomokit/geometry.py); the conventions are the
reference's (geometry.py:3-16):

* right-handed world, rotation axis +z, isocentre at the origin;
* trajectory angle 0 puts the source on +x, rotation is counter-clockwise;
* the detector v axis points along +z, u is tangent to the orbit;
* ``P @ (x, 1) = (w*col, w*row, w)`` with the principal point at the detector
  centre pixel and the third row a unit vector (``w`` = metric depth).

What is new here: pose lists are converted to matrices in one vectorised pass;
geometries cache the per-view arrays the kernels consume (angles as cos/sin,
the (V,3,4) matrix stack, sources and M^-1) so repeated operator calls do no
host work; helical and sinusoidal trajectory builders; and a PYRO-NN style
``Geometry`` front end (``init_from_parameters`` / ``set_trajectory``).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from functools import cached_property
from pathlib import Path
from typing import Iterable

import numpy as np

__all__ = [
    "DegeneratePoseError",
    "Pose",
    "ProjectionMatrix",
    "GeometryParallel2D",
    "GeometryFan2D",
    "GeometryCone3D",
    "Geometry",
    "circular_trajectory_2d",
    "circular_pose",
    "pose_to_projection_matrix",
    "poses_to_matrix_array",
    "circular_trajectory_3d",
    "helical_trajectory_3d",
    "sinusoidal_trajectory_3d",
    "trajectory_from_poses",
    "load_projection_matrices",
    "save_projection_matrices",
    "circular_cone_geometry",
]

_TOL = 1e-9  # reference _UNIT_TOL (geometry.py:43)


class DegeneratePoseError(ValueError):
    """A pose whose rays run parallel to the detector plane (no pinhole map)."""


def _vec3(value, name: str) -> np.ndarray:
    v = np.asarray(value, dtype=np.float64).reshape(-1)
    if v.shape != (3,):
        raise ValueError(f"{name} must be a 3-vector")
    return v


def _frozen(arr: np.ndarray) -> np.ndarray:
    arr = np.array(arr, dtype=np.float64, copy=True)
    arr.setflags(write=False)
    return arr


# ---------------------------------------------------------------------------
# poses and matrices
# ---------------------------------------------------------------------------


@dataclass(frozen=True, eq=False)
class Pose:
    """Source and detector placement of one view (geometry.py:57-99).

    ``u_dir`` is the detector column axis and ``v_dir`` the row axis: unit,
    orthogonal, with the source off the detector plane.
    """

    source_position: np.ndarray
    detector_center: np.ndarray
    u_dir: np.ndarray
    v_dir: np.ndarray

    def __post_init__(self):
        src = _vec3(self.source_position, "source_position")
        ctr = _vec3(self.detector_center, "detector_center")
        u = _vec3(self.u_dir, "u_dir")
        v = _vec3(self.v_dir, "v_dir")
        if abs(float(np.linalg.norm(u)) - 1.0) > _TOL:
            raise ValueError("u_dir must be unit length")
        if abs(float(np.linalg.norm(v)) - 1.0) > _TOL:
            raise ValueError("v_dir must be unit length")
        if abs(float(u @ v)) > _TOL:
            raise ValueError("u_dir and v_dir must be orthogonal")
        if abs(float((ctr - src) @ np.cross(u, v))) <= _TOL:
            raise ValueError("source must lie off the detector plane")
        for name, arr in (("source_position", src), ("detector_center", ctr), ("u_dir", u),
                          ("v_dir", v)):
            object.__setattr__(self, name, _frozen(arr))

    @property
    def normal(self) -> np.ndarray:
        """Detector normal oriented from the source toward the detector plane."""
        n = np.cross(self.u_dir, self.v_dir)
        return -n if float((self.detector_center - self.source_position) @ n) < 0 else n


@dataclass(frozen=True, eq=False)
class ProjectionMatrix:
    """Normalised 3x4 world -> homogeneous detector-pixel map (geometry.py:102-145)."""

    entries: np.ndarray

    def __post_init__(self):
        m = np.asarray(self.entries, dtype=np.float64).reshape(3, 4)
        scale = max(1.0, float(np.abs(m).max()))
        if np.linalg.matrix_rank(m, tol=1e-9 * scale) < 3:
            raise ValueError("projection matrix must have rank 3")
        if abs(float(np.linalg.norm(m[2, :3])) - 1.0) > 1e-6:
            raise ValueError("third-row direction must be unit (normalized form)")
        object.__setattr__(self, "entries", _frozen(m))

    @classmethod
    def from_raw(cls, entries) -> "ProjectionMatrix":
        """Normalise any homogeneous representative: divide by the third-row
        direction norm, signed so that the isocentre depth P[2,3] is positive."""
        m = np.asarray(entries, dtype=np.float64).reshape(3, 4)
        k = float(np.linalg.norm(m[2, :3]))
        if k == 0.0:
            raise ValueError("third row direction must be nonzero")
        return cls(m / (-k if m[2, 3] < 0 else k))

    def source_position(self) -> np.ndarray:
        """Centre of projection = right null vector of P, dehomogenised."""
        h = np.linalg.svd(self.entries)[2][-1]
        if abs(h[3]) < 1e-300:
            raise ValueError("projection center at infinity")
        return h[:3] / h[3]

    def project(self, points) -> np.ndarray:
        """World points (..., 3) -> pixel (col, row) (..., 2)."""
        pts = np.asarray(points, dtype=np.float64)
        hom = pts @ self.entries[:, :3].T + self.entries[:, 3]
        return hom[..., :2] / hom[..., 2:3]


def _detector_args(detector_shape, detector_spacing):
    rows, cols = (int(n) for n in detector_shape)
    dv, du = (float(s) for s in detector_spacing)
    if rows < 1 or cols < 1 or du <= 0 or dv <= 0:
        raise ValueError("invalid detector shape/spacing")
    return rows, cols, dv, du


def poses_to_matrix_array(sources, centers, u_dirs, v_dirs, detector_shape,
                          detector_spacing) -> np.ndarray:
    """Vectorised pinhole maps of V poses -> (V, 3, 4) float64.

    Row construction of geometry.py:273-280: with depth D = (c - s).n,
    P0 = (D/du) u + (c_u - (c-s).u/du) n, P1 = (D/dv) v + (c_v - (c-s).v/dv) n,
    P2 = n, and P[:, 3] = -P[:, :3] s.
    """
    rows, cols, dv, du = _detector_args(detector_shape, detector_spacing)
    s = np.asarray(sources, dtype=np.float64).reshape(-1, 3)
    c = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
    u = np.asarray(u_dirs, dtype=np.float64).reshape(-1, 3)
    v = np.asarray(v_dirs, dtype=np.float64).reshape(-1, 3)
    off = c - s
    n = np.cross(u, v)
    n = np.where((np.einsum("ij,ij->i", off, n) < 0)[:, None], -n, n)
    depth = np.einsum("ij,ij->i", off, n)
    bad = np.flatnonzero(np.abs(depth) <= _TOL)
    if bad.size:
        raise DegeneratePoseError(f"pose {int(bad[0])}: central ray parallel to detector plane")
    cu, cv = (cols - 1) / 2.0, (rows - 1) / 2.0
    m = np.empty((s.shape[0], 3, 4))
    m[:, 0, :3] = (depth / du)[:, None] * u + (cu - np.einsum("ij,ij->i", off, u) / du)[:, None] * n
    m[:, 1, :3] = (depth / dv)[:, None] * v + (cv - np.einsum("ij,ij->i", off, v) / dv)[:, None] * n
    m[:, 2, :3] = n
    m[:, :, 3] = -np.einsum("vij,vj->vi", m[:, :, :3], s)
    return m


def pose_to_projection_matrix(pose: Pose, detector_shape, detector_spacing) -> ProjectionMatrix:
    """Pinhole map of one pose (geometry.py:251-281)."""
    _detector_args(detector_shape, detector_spacing)
    depth = float((pose.detector_center - pose.source_position) @ pose.normal)
    if abs(depth) <= _TOL:
        raise DegeneratePoseError("central ray parallel to detector plane")
    m = poses_to_matrix_array(pose.source_position, pose.detector_center, pose.u_dir, pose.v_dir,
                              detector_shape, detector_spacing)[0]
    return ProjectionMatrix(m)


def circular_trajectory_2d(n_projections: int, angular_range: float) -> np.ndarray:
    """Equispaced angles i * range / n, i = 0..n-1 (geometry.py:240-248)."""
    n = int(n_projections)
    if n < 1:
        raise ValueError("n_projections must be >= 1")
    span = float(angular_range)
    if span <= 0:
        raise ValueError("angular_range must be positive")
    return np.arange(n) * (span / n)


def circular_pose(theta: float, sdd: float, sid: float) -> Pose:
    """Pose of the circular orbit at angle theta (geometry.py:284-292)."""
    ct, st = math.cos(theta), math.sin(theta)
    return Pose(np.array([sid * ct, sid * st, 0.0]),
                np.array([-(sdd - sid) * ct, -(sdd - sid) * st, 0.0]),
                np.array([-st, ct, 0.0]), np.array([0.0, 0.0, 1.0]))


def _orbit_frames(theta: np.ndarray, sdd: float, sid: float, z: np.ndarray):
    """Vectorised circular-orbit frames with the source and detector centre
    lifted to height z (u tangent, v = +z)."""
    ct, st = np.cos(theta), np.sin(theta)
    zeros = np.zeros_like(theta)
    src = np.stack([sid * ct, sid * st, z], axis=1)
    ctr = np.stack([-(sdd - sid) * ct, -(sdd - sid) * st, z], axis=1)
    u = np.stack([-st, ct, zeros], axis=1)
    v = np.tile([0.0, 0.0, 1.0], (theta.size, 1))
    return src, ctr, u, v


def _check_distances(sdd, sid):
    sdd, sid = float(sdd), float(sid)
    if not 0.0 < sid < sdd:
        raise ValueError("requires 0 < sid < sdd")
    return sdd, sid


def _as_matrices(arr: np.ndarray) -> list[ProjectionMatrix]:
    return [ProjectionMatrix(m) for m in arr]


def circular_trajectory_3d(n_projections=None, angular_range=None, sdd=None, sid=None,
                           detector_shape=None, detector_spacing=None,
                           **params) -> list[ProjectionMatrix]:
    """Matrices of the closed-form circular orbit (geometry.py:295-312).

    Also accepts the PYRO-NN parameter dict (``number_of_projections``, ...)
    as keyword arguments, as in the paper's Listing 1.
    """
    n = n_projections if n_projections is not None else params.get("number_of_projections")
    sdd = sdd if sdd is not None else params.get("source_detector_distance")
    sid = sid if sid is not None else params.get("source_isocenter_distance")
    sdd, sid = _check_distances(sdd, sid)
    theta = circular_trajectory_2d(n, angular_range)
    frames = _orbit_frames(theta, sdd, sid, np.zeros_like(theta))
    return _as_matrices(poses_to_matrix_array(*frames, detector_shape, detector_spacing))


def helical_trajectory_3d(n_projections: int, angular_range: float, sdd: float, sid: float,
                          detector_shape, detector_spacing, z_start: float,
                          z_end: float) -> list[ProjectionMatrix]:
    """Helix: source (sid cos t, sid sin t, z(t)), detector centre at the same
    height, z rising linearly from z_start to z_end over the angular range
    (endpoint excluded, like the circular orbit)."""
    sdd, sid = _check_distances(sdd, sid)
    theta = circular_trajectory_2d(n_projections, angular_range)
    z = float(z_start) + (float(z_end) - float(z_start)) * theta / float(angular_range)
    frames = _orbit_frames(theta, sdd, sid, z)
    return _as_matrices(poses_to_matrix_array(*frames, detector_shape, detector_spacing))


def sinusoidal_trajectory_3d(n_projections: int, angular_range: float, sdd: float, sid: float,
                             detector_shape, detector_spacing, amplitude: float,
                             frequency: float = 2.0) -> list[ProjectionMatrix]:
    """Sinusoidal orbit: z(t) = amplitude * sin(frequency * t)."""
    sdd, sid = _check_distances(sdd, sid)
    theta = circular_trajectory_2d(n_projections, angular_range)
    frames = _orbit_frames(theta, sdd, sid, float(amplitude) * np.sin(float(frequency) * theta))
    return _as_matrices(poses_to_matrix_array(*frames, detector_shape, detector_spacing))


def trajectory_from_poses(poses: Iterable[Pose], detector_shape,
                          detector_spacing) -> list[ProjectionMatrix]:
    """Pose-wise pinhole maps, order preserved (geometry.py:315-328)."""
    poses = list(poses)
    if not poses:
        raise ValueError("at least one pose required")
    try:
        _detector_args(detector_shape, detector_spacing)
    except ValueError as exc:
        raise DegeneratePoseError(f"pose 0: {exc}") from exc
    arr = poses_to_matrix_array([p.source_position for p in poses],
                                [p.detector_center for p in poses],
                                [p.u_dir for p in poses], [p.v_dir for p in poses],
                                detector_shape, detector_spacing)
    out = []
    for i, m in enumerate(arr):
        try:
            out.append(ProjectionMatrix(m))
        except ValueError as exc:
            raise DegeneratePoseError(f"pose {i}: {exc}") from exc
    return out


def load_projection_matrices(path) -> list[ProjectionMatrix]:
    """Read ``{"matrices": [[12 row-major numbers], ...]}`` and renormalise."""
    p = Path(path)
    try:
        doc = json.loads(p.read_text())
    except json.JSONDecodeError as exc:
        raise ValueError(f"malformed matrix file {p}: {exc}") from exc
    if not isinstance(doc, dict) or "matrices" not in doc:
        raise ValueError(f"matrix file {p} must contain a 'matrices' list")
    mats = []
    for i, flat in enumerate(doc["matrices"]):
        arr = np.asarray(flat, dtype=np.float64).reshape(-1)
        if arr.size != 12:
            raise ValueError(f"matrix {i}: expected 12 entries, got {arr.size}")
        mats.append(ProjectionMatrix.from_raw(arr.reshape(3, 4)))
    if not mats:
        raise ValueError(f"matrix file {p} holds no matrices")
    return mats


def save_projection_matrices(matrices, path) -> None:
    """Write matrices in the JSON exchange format read by the loader."""
    doc = {"matrices": [[float(x) for x in np.asarray(m.entries).ravel()] for m in matrices]}
    Path(path).write_text(json.dumps(doc, indent=2) + "\n")


# ---------------------------------------------------------------------------
# beam geometries
# ---------------------------------------------------------------------------


@dataclass(frozen=True, eq=False)
class GeometryParallel2D:
    """Parallel-beam fan of rays per angle (geometry.py:148-177)."""

    volume_shape: tuple
    volume_spacing: tuple
    detector_width: int
    detector_spacing: float
    angles: np.ndarray

    def __post_init__(self):
        ang = np.asarray(self.angles, dtype=np.float64).reshape(-1)
        if ang.size < 1:
            raise ValueError("at least one projection angle required")
        if not np.isfinite(ang).all():
            raise ValueError("angles must be finite")
        object.__setattr__(self, "angles", _frozen(ang))
        msg = "parallel geometry references a 2D volume"
        object.__setattr__(self, "volume_shape", tuple(int(n) for n in self.volume_shape))
        object.__setattr__(self, "volume_spacing", tuple(float(x) for x in self.volume_spacing))
        object.__setattr__(self, "detector_width", int(self.detector_width))
        object.__setattr__(self, "detector_spacing", float(self.detector_spacing))
        if len(self.volume_shape) != 2 or len(self.volume_spacing) != 2:
            raise ValueError(msg)
        if self.detector_width < 1 or self.detector_spacing <= 0:
            raise ValueError("invalid detector parameters")

    @property
    def n_projections(self) -> int:
        return int(self.angles.size)

    @property
    def sinogram_shape(self) -> tuple:
        return (self.n_projections, self.detector_width)

    @cached_property
    def trig(self) -> tuple:
        """(cos, sin) of the angles as contiguous float64 arrays (kernel input)."""
        return (np.ascontiguousarray(np.cos(self.angles)), np.ascontiguousarray(np.sin(self.angles)))


@dataclass(frozen=True, eq=False)
class GeometryFan2D(GeometryParallel2D):
    """Fan beam from a point source at sid, flat detector at sdd (geometry.py:180-190)."""

    sdd: float = 0.0
    sid: float = 0.0

    def __post_init__(self):
        super().__post_init__()
        object.__setattr__(self, "sdd", float(self.sdd))
        object.__setattr__(self, "sid", float(self.sid))
        if not 0.0 < self.sid < self.sdd:
            raise ValueError("fan geometry requires 0 < sid < sdd")


@dataclass(frozen=True, eq=False)
class GeometryCone3D:
    """Cone beam: one projection matrix per view (geometry.py:193-237).

    ``detector_shape`` is (rows, cols), ``detector_spacing`` (dv, du); sdd/sid
    are kept for the reconstruction weights.  For PYRO-NN style construction
    (Listing 1) ``matrices`` may be omitted and ``number_of_projections`` /
    ``angular_range`` given instead: the circular orbit is then built.
    """

    volume_shape: tuple
    volume_spacing: tuple
    detector_shape: tuple
    detector_spacing: tuple
    matrices: tuple = None
    sdd: float = None
    sid: float = None
    number_of_projections: int | None = field(default=None, repr=False)
    angular_range: float | None = field(default=None, repr=False)

    def __post_init__(self):
        object.__setattr__(self, "volume_shape", tuple(int(n) for n in self.volume_shape))
        object.__setattr__(self, "volume_spacing", tuple(float(s) for s in self.volume_spacing))
        object.__setattr__(self, "detector_shape", tuple(int(n) for n in self.detector_shape))
        object.__setattr__(self, "detector_spacing", tuple(float(s) for s in self.detector_spacing))
        if self.sdd is None or self.sid is None:
            raise ValueError("cone geometry requires 0 < sid < sdd")
        object.__setattr__(self, "sdd", float(self.sdd))
        object.__setattr__(self, "sid", float(self.sid))
        if len(self.volume_shape) != 3 or len(self.volume_spacing) != 3:
            raise ValueError("cone geometry references a 3D volume")
        if len(self.detector_shape) != 2 or len(self.detector_spacing) != 2:
            raise ValueError("cone detector is 2D (rows, cols)")
        if not 0.0 < self.sid < self.sdd:
            raise ValueError("cone geometry requires 0 < sid < sdd")
        mats = self.matrices
        if mats is None and self.number_of_projections is not None:
            mats = circular_trajectory_3d(self.number_of_projections,
                                          self.angular_range if self.angular_range else 2 * math.pi,
                                          self.sdd, self.sid, self.detector_shape,
                                          self.detector_spacing)
        mats = tuple(mats) if mats is not None else ()
        if not mats:
            raise ValueError("at least one projection matrix required")
        if not all(isinstance(m, ProjectionMatrix) for m in mats):
            raise ValueError("matrices must be ProjectionMatrix instances")
        object.__setattr__(self, "matrices", mats)

    @property
    def n_projections(self) -> int:
        return len(self.matrices)

    @property
    def sinogram_shape(self) -> tuple:
        return (self.n_projections, *self.detector_shape)

    def matrix_array(self) -> np.ndarray:
        return self._matrix_stack

    @cached_property
    def _matrix_stack(self) -> np.ndarray:
        arr = np.ascontiguousarray(np.stack([m.entries for m in self.matrices]))
        arr.setflags(write=False)
        return arr

    @cached_property
    def ray_constants(self) -> tuple:
        """(sources (V,3), M^-1 (V,3,3)) for the ray-driven projector
        (projectors.py:191-202: singular M rejected, source = SVD null vector)."""
        mats = self._matrix_stack
        blocks = mats[:, :, :3]
        det = np.linalg.det(blocks)
        bad = np.flatnonzero(np.abs(det) < 1e-12)
        if bad.size:
            raise ValueError(f"projection matrix {int(bad[0])} is degenerate (singular M block)")
        h = np.linalg.svd(mats)[2][:, -1, :]
        if np.any(np.abs(h[:, 3]) < 1e-300):
            raise ValueError("projection center at infinity")
        sources = np.ascontiguousarray(h[:, :3] / h[:, 3:4])
        minv = np.ascontiguousarray(np.linalg.inv(blocks))
        return sources, minv

    def set_trajectory(self, matrices) -> "GeometryCone3D":
        """PYRO-NN style: replace the trajectory (matrices or a (V,3,4) array)."""
        mats = [m if isinstance(m, ProjectionMatrix) else ProjectionMatrix(m) for m in matrices]
        if not mats:
            raise ValueError("at least one projection matrix required")
        object.__setattr__(self, "matrices", tuple(mats))
        for key in ("_matrix_stack", "ray_constants"):
            self.__dict__.pop(key, None)
        return self


def circular_cone_geometry(volume_shape, volume_spacing, detector_shape, detector_spacing,
                           number_of_projections, angular_range, sdd, sid) -> GeometryCone3D:
    """Circular-orbit cone geometry from scan parameters (geometry.py:357-379)."""
    return GeometryCone3D(volume_shape, volume_spacing, detector_shape, detector_spacing,
                          circular_trajectory_3d(number_of_projections, angular_range, sdd, sid,
                                                 detector_shape, detector_spacing), sdd, sid)


class Geometry:
    """PYRO-NN style geometry front end.

    ``Geometry().init_from_parameters(...)`` records the scan parameters; the
    ``parallel2d`` / ``fan2d`` / ``cone3d`` properties (or ``build()``) return
    the typed geometry the operators consume.  ``set_trajectory`` installs
    projection matrices (cone) or angles (2D).
    """

    def __init__(self):
        self.params: dict = {}
        self._trajectory = None

    def init_from_parameters(self, volume_shape, volume_spacing, detector_shape,
                             detector_spacing, number_of_projections, angular_range,
                             trajectory=None, source_isocenter_distance=None,
                             source_detector_distance=None, **extra) -> "Geometry":
        sid = source_isocenter_distance if source_isocenter_distance is not None else extra.get("sid")
        sdd = source_detector_distance if source_detector_distance is not None else extra.get("sdd")
        self.params = dict(volume_shape=tuple(volume_shape), volume_spacing=tuple(volume_spacing),
                           detector_shape=tuple(np.atleast_1d(detector_shape)),
                           detector_spacing=tuple(np.atleast_1d(detector_spacing)),
                           number_of_projections=int(number_of_projections),
                           angular_range=float(angular_range), sid=sid, sdd=sdd)
        if trajectory is not None:
            self.set_trajectory(trajectory if not callable(trajectory) else trajectory(**self.params))
        return self

    def set_trajectory(self, trajectory) -> "Geometry":
        self._trajectory = trajectory
        return self

    @property
    def kind(self) -> str:
        if len(self.params["volume_shape"]) == 3:
            return "cone3d"
        return "fan2d" if self.params.get("sdd") else "parallel2d"

    def build(self):
        p = self.params
        if self.kind == "cone3d":
            traj = self._trajectory
            if traj is None:
                traj = circular_trajectory_3d(p["number_of_projections"], p["angular_range"], p["sdd"],
                                              p["sid"], p["detector_shape"], p["detector_spacing"])
            mats = [m if isinstance(m, ProjectionMatrix) else ProjectionMatrix(m) for m in traj]
            return GeometryCone3D(p["volume_shape"], p["volume_spacing"], p["detector_shape"],
                                  p["detector_spacing"], mats, p["sdd"], p["sid"])
        angles = (np.asarray(self._trajectory, dtype=np.float64) if self._trajectory is not None
                  else circular_trajectory_2d(p["number_of_projections"], p["angular_range"]))
        if self.kind == "fan2d":
            return GeometryFan2D(p["volume_shape"], p["volume_spacing"], p["detector_shape"][0],
                                 p["detector_spacing"][0], angles, sdd=p["sdd"], sid=p["sid"])
        return GeometryParallel2D(p["volume_shape"], p["volume_spacing"], p["detector_shape"][0],
                                  p["detector_spacing"][0], angles)

    parallel2d = property(build)
    fan2d = property(build)
    cone3d = property(build)
