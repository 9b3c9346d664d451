"""Analytic backward: pixel gradients -> every learnable cloud field.

Mirrors ``render_backward`` (``pkg/src/xsplat/rasterizer/backward.py:21-124``):
stale-splat and shape checks, then the reverse replay of the compositing
(K4a, ``xg_composite_bwd``) and the per-Gaussian chain rule through the
conic inverse, the projected covariance (including the Jacobian's own
dependence on the camera-space mean), R S S^T R^T, the quaternion
normalisation and both sigmoids (K4b, ``xg_preprocess_bwd``).
"""

from __future__ import annotations

import torch

from .. import _native as nat
from ..errors import InvalidParameterError, StaleSplatsError
from ..gaussians import GaussianCloud, flat_views
from .frontend import RenderGradients, SplatList


def make_gradients(n: int, n_features: int, device) -> RenderGradients:
    flat = torch.empty(n * (11 + n_features), dtype=torch.float32, device=device)
    v = flat_views(flat, n, n_features)
    return RenderGradients(
        positions=v["positions"],
        rotations=v["rotations"],
        log_scales=v["log_scales"],
        raw_opacities=v["raw_opacities"],
        features=v["features"],
        screen_norms=torch.empty(n, dtype=torch.float32, device=device),
        visible=torch.empty(n, dtype=torch.bool, device=device),
        flat=flat,
    )


def render_backward(cloud: GaussianCloud, splats: SplatList, dl_dimage, kernel_grads: dict | None = None
                    ) -> RenderGradients:
    """Exact gradients of the loss w.r.t. every learnable attribute.

    ``kernel_grads`` (optional dict of float64 [N,2]/[N,3]/[N]/[N] tensors
    ``g_mean``, ``g_conic``, ``g_int``, ``g_alpha``) additionally receives the
    reference's kernel-level gradients (``backward_tiles`` outputs).
    """
    if cloud.fingerprint() != splats.cloud_fingerprint:
        raise StaleSplatsError("cloud was mutated after the forward render; re-render before backward")
    h, w = splats.image_shape
    if not isinstance(dl_dimage, torch.Tensor):
        dl_dimage = torch.as_tensor(dl_dimage)
    if tuple(dl_dimage.shape) != (h, w):
        raise InvalidParameterError(f"pixel gradient shape {tuple(dl_dimage.shape)} != image shape {(h, w)}")
    dl = dl_dimage.to(device=cloud.device, dtype=torch.float32).contiguous()
    frame = splats.frame
    n = cloud.n_points
    grads = make_gradients(n, cloud.n_features, cloud.device)
    if not frame.has_forward:
        frame.composite()
    acc = torch.empty((n, 8), dtype=torch.float32, device=cloud.device)
    vis = torch.empty(n, dtype=torch.uint8, device=cloud.device)
    frame.backward(cloud, acc, grads.flat, grads.screen_norms, vis, dl_dimage=dl,
                   kernel_grads=kernel_grads)
    grads.visible = vis.bool()
    return grads
