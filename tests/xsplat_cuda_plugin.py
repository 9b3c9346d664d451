"""pytest plugin (``-p xsplat_cuda_plugin``) for running xsplat's OWN test
modules against the engine: registers the ``"cuda"`` kernel backend
(paper_2403_04116_b200/rasterizer/xsplat_backend.py) in the imported
reference's registry before collection, so every test that takes the
``backend`` fixture (test_rasterizer.py:26-36, parametrised over
available_backends()) also runs on it; with XSPLAT_CUDA_ACTIVE=1 it is made
the active backend for the whole session (test_gradients.py uses the
active one)."""

import os


def pytest_configure(config):
    import torch

    torch.cuda.set_device(0)
    from xsplat.rasterizer import backend

    from paper_2403_04116_b200.rasterizer import xsplat_backend

    xsplat_backend.register(backend)
    if os.environ.get("XSPLAT_CUDA_ACTIVE") == "1":
        backend.set_backend("cuda")
