"""B200-native Differentiable Radiative Rasterization (X-Gaussian, arXiv 2403.04116).

A drop-in for the reference engine's hot path (``xsplat``): the same Python
API - ``GaussianCloud``, ``render`` / ``render_view`` / ``project_splats`` /
``render_backward``, ``adam_step`` / ``densify_and_prune`` / ``train`` - on
hand-written sm_100a CUDA kernels behind the C ABI of ``include/xgauss.h``
(libxgauss.so) - plus the path's callers on either side: the SSIM loss
(``metrics``), the cone-beam phantom projector that makes training targets
(``phantom``, ``dataset``).  There is no CPU fallback.
"""

import os as _os

# The sweep renderer keeps ~14 streams busy (12 binning streams, compositing,
# image downloads); with CUDA's default 8 hardware work queues some of them
# share a queue and serialise (a download then holds up a binning chain).
# 32 queues: C3 sweep +1.5 % device-resident and end to end (measured,
# DESIGN.md).  Read when the CUDA context is created, so it only applies if
# the package is imported before CUDA is initialised; an explicit setting wins.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .acui import CuboidSpec, init_alternative, init_cloud, sample_cuboid
from .dataset import ProjectionSet, add_noise, load_dataset, make_projection_set, save_dataset
from .errors import (
    ConfigError,
    DatasetError,
    InvalidParameterError,
    NativeError,
    NumericalDegeneracyError,
    StaleSplatsError,
    TooManyPointsError,
    TrainingDivergenceError,
    XSplatError,
)
from .gaussians import (
    GaussianCloud,
    RadiativeGaussian,
    covariance_2d,
    covariance_3d,
    logit,
    quaternions_to_rotations,
    rirf,
    sigmoid,
)
from .geometry import (
    ExtrinsicMatrix,
    IntrinsicMatrix,
    ScannerConfig,
    camera_to_image,
    equal_interval_angles,
    extrinsic_from_angle,
    intrinsic_from_config,
    projection_jacobian,
    viewing_rotation,
    world_to_camera,
)
from .metrics import MetricReport, psnr, ssim, ssim_and_gradient
from .phantom import (
    Cuboid,
    Ellipsoid,
    VoxelPhantom,
    default_phantom_primitives,
    make_phantom,
    primitive_from_dict,
    project_all,
    project_phantom,
)
from .rasterizer import (
    Projection,
    RenderGradients,
    SplatList,
    active_backend,
    blend_pixel,
    brute_force_render,
    project_splats,
    render,
    render_backward,
    render_view,
)

__version__ = "0.1.0"
