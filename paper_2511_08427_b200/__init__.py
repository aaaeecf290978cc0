"""B200-native (sm_100a) differentiable CT operators.

Drop-in for the projector hot path of the reference (tomokit, the CPU
re-implementation of PYRO-NN, arXiv 2511.08427): ray-driven forward and
voxel-driven back projectors for parallel 2D, fan 2D and cone 3D, their
autograd adjoint pairs, and the FBP/FDK pipeline -- on CUDA tensors, executed
by hand-written sm_100a kernels in libtkb200.so (C ABI: include/tk_b200.h).

Names follow the reference (``tomokit`` functions, the ``tomokit_layers``
``py_*`` boundary) and PYRO-NN (``ConeProjection3D``, ``Geometry``,
``shepp_logan_3D``, ``fft_and_ifft``).
"""

from .autodiff import (DifferentiableOp, GradCheckReport, back_projection_op, dot_test, fbp_op,
                       fft_filter_op, forward_projection_op, grad_check, vjp_back_projection,
                       vjp_fft_filter, vjp_forward_projection)
from .config import ConfigError, PipelineConfig, load_config
from .filters import (Filter1D, backproject_stage, cosine_3D, cosine_filter, cosine_preweight_cone,
                      fbp_fan_2d, fbp_parallel_2d, fdk_cone_3d, fdk_tensor, fft_and_ifft,
                      fft_filter, filter_stage, ramp_3D, ramp_filter, reconstruction_filter,
                      shepp_logan_3D, shepp_logan_filter)
from .geometry import (DegeneratePoseError, Geometry, GeometryCone3D, GeometryFan2D,
                       GeometryParallel2D, Pose, ProjectionMatrix, circular_cone_geometry,
                       circular_pose, circular_trajectory_2d, circular_trajectory_3d,
                       helical_trajectory_3d, load_projection_matrices, pose_to_projection_matrix,
                       save_projection_matrices, sinusoidal_trajectory_3d, trajectory_from_poses)
from .grids import (GridFormatError, Sinogram, SizeMismatchError, UnsupportedDtypeError, Volume,
                    read_grid, write_grid)
from .layers import (ConeBackProjection3D, ConeBackProjectionFor3D, ConeProjection3D,
                     ConeProjectionFor3D, FanBackProjection2D, FanBackProjectionFor2D,
                     FanProjection2D, FanProjectionFor2D, ParallelBackProjection2D,
                     ParallelBackProjectionFor2D, ParallelProjection2D, ParallelProjectionFor2D)
from .projectors import (SamplingConfig, back_project, back_project_cone_3d, back_project_fan_2d,
                         back_project_parallel_2d, forward_project, forward_project_cone_3d,
                         forward_project_fan_2d, forward_project_parallel_2d, materialize_operator,
                         transpose_back_project, transpose_forward_project)

from . import phantoms  # noqa: E402  (synthetic inputs on the GPU)
from . import artifacts  # noqa: E402  (sinogram degradation simulators, reference artifacts.py)
from .artifacts import (add_detector_jitter, add_gantry_motion_blur, add_gaussian_noise,  # noqa: E402
                        add_poisson_noise, add_ring_artifact)

__version__ = "0.1.0"
