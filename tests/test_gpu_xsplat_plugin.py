"""The drop-in proof inside the REAL xsplat: the engine registered as
xsplat's ``"cuda"`` kernel backend (rasterizer/backend.py:20-46, the
reference's own plug-in point; paper_2403_04116_b200/rasterizer/
xsplat_backend.py) and xsplat's own test modules run against it - the
reference built into oracle/_ref by oracle/build_ref.sh, its tests copied
next to it (oracle/_ref/xsplat_tests, git-ignored like the build).

* test_rasterizer.py with "cuda" registered: every backend-parametrised
  test gets a [cuda] case (test_rasterizer.py:26-36) and passes.  Only
  three tests fail, by construction: they hard-code a two-entry registry
  (TestBackendLockstep unpacks exactly two backends;
  test_unknown_backend_rejected expects "cuda" to be unknown).
* test_gradients.py with "cuda" the ACTIVE backend: finite differences at
  rel 1e-3 on every element of every field and the closed forms at rel
  1e-12 / 1e-10 all pass.
* the lockstep check the reference runs between its two backends
  (test_rasterizer.py:223-257), cuda vs compiled, at the reference's own
  tolerances (images rtol 1e-12, gradients rtol 1e-9 + 1e-12 of the max),
  through xsplat's render / render_backward on the reference's seeded
  scenes.

The backend is xg_forward_tiles_f64 / xg_backward_tiles_f64: float64 in the
Cython loop's operation order (csrc/xg_tiles64.cu).
"""

from __future__ import annotations

import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"
REF_TESTS = REF / "xsplat_tests"

EXPECTED_RASTERIZER = {
    "test_forward_agreement",        # TestBackendLockstep: unpacks exactly two backends
    "test_backward_agreement",       # (same)
    "test_unknown_backend_rejected",  # expects "cuda" to be unregistered
}


def _have_ref() -> bool:
    return (REF / "xsplat" / "rasterizer").is_dir() and REF_TESTS.is_dir()


def _run(module: str, active: bool, tmp_path) -> dict:
    xml = tmp_path / f"{module}.xml"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests"), env.get("PYTHONPATH", "")])
    env["XSPLAT_CUDA_ACTIVE"] = "1" if active else "0"
    proc = subprocess.run([sys.executable, "-m", "pytest", str(REF_TESTS / module), "-p", "xsplat_cuda_plugin",
                           "-q", "-p", "no:cacheprovider", f"--junitxml={xml}", "--rootdir", str(REF_TESTS)],
                          cwd=str(REF_TESTS), env=env, capture_output=True, text=True, timeout=1200)
    assert xml.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    out = {}
    for case in ET.parse(xml).getroot().iter("testcase"):
        name = case.get("name")
        status = "passed"
        for child in case:
            if child.tag in ("failure", "error"):
                status = "failed"
            elif child.tag == "skipped":
                status = "skipped"
        out[f"{case.get('classname')}::{name}"] = (name, status)
    print(f"\n[{module}] {sum(s == 'passed' for _, s in out.values())} passed, "
          f"{sum(s == 'failed' for _, s in out.values())} failed, "
          f"{sum(s == 'skipped' for _, s in out.values())} skipped")
    return out


@pytest.mark.skipif(not _have_ref(), reason="oracle/_ref (oracle/build_ref.sh) not built")
def test_reference_rasterizer_suite_with_cuda_backend(tmp_path):
    res = _run("test_rasterizer.py", False, tmp_path)
    cuda_cases = [k for k, (n, _) in res.items() if n.endswith("[cuda]")]
    assert len(cuda_cases) >= 14, cuda_cases
    failed = {n for n, s in res.values() if s == "failed"}
    print("  failed:", sorted(failed))
    assert failed <= EXPECTED_RASTERIZER, failed - EXPECTED_RASTERIZER
    assert all(res[k][1] == "passed" for k in cuda_cases), [k for k in cuda_cases if res[k][1] != "passed"]


@pytest.mark.skipif(not _have_ref(), reason="oracle/_ref (oracle/build_ref.sh) not built")
def test_reference_gradient_suite_on_cuda_backend(tmp_path):
    res = _run("test_gradients.py", True, tmp_path)
    failed = {n for n, s in res.values() if s != "passed"}
    print("  not passed:", sorted(failed))
    assert not failed and len(res) >= 10, failed


@pytest.mark.skipif(not _have_ref(), reason="oracle/_ref (oracle/build_ref.sh) not built")
def test_lockstep_cuda_vs_compiled():
    """test_rasterizer.py:223-257's backend lockstep, cuda against compiled,
    at the reference's tolerances: images rtol 1e-12 (atol 1e-14),
    gradients rtol 1e-9 (atol 1e-12 of the field's max)."""
    import importlib.util

    import torch

    torch.cuda.set_device(0)
    sys.path.insert(0, str(REF))
    spec = importlib.util.spec_from_file_location("xsplat_ref_conftest", REF_TESTS / "conftest.py")
    ref_conftest = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ref_conftest)  # the reference's own fixtures (conftest.py:8-45)
    from xsplat.rasterizer import backend, render_backward, render_view

    from paper_2403_04116_b200.rasterizer import xsplat_backend

    xsplat_backend.register(backend)
    previous = backend.active_backend()
    rng = np.random.default_rng(1234)
    worst_img = worst_grad = 0.0
    try:
        for trial in range(12):
            sc = ref_conftest.small_scanner(width=32, height=32, pitch=6.0)
            cloud = ref_conftest.random_cloud(int(rng.integers(4, 24)), rng, pos_scale=30.0)
            phi = float(rng.uniform(0, np.pi))
            up = rng.normal(size=(32, 32))
            res = {}
            for name in ("compiled", "cuda"):
                backend.set_backend(name)
                proj, sp = render_view(cloud, sc, phi)
                res[name] = (proj.pixels, render_backward(cloud, sp, up))
            a, b = res["compiled"][0], res["cuda"][0]
            assert np.allclose(b, a, rtol=1e-12, atol=1e-14), trial
            worst_img = max(worst_img, float((np.abs(a - b) / np.maximum(np.abs(a), 1e-300)).max()))
            ga, gb = res["compiled"][1], res["cuda"][1]
            for f in ("positions", "rotations", "log_scales", "raw_opacities", "features", "screen_norms"):
                x, y = getattr(ga, f), getattr(gb, f)
                scale = max(float(np.abs(x).max()), 1e-300)
                assert np.allclose(y, x, rtol=1e-9, atol=1e-12 * scale), (trial, f)
                worst_grad = max(worst_grad, float(np.abs(x - y).max() / scale))
            assert np.array_equal(ga.visible, gb.visible), trial
    finally:
        backend.set_backend(previous)
        backend._BACKENDS.pop("cuda", None)
    print(f"\nlockstep cuda vs compiled: image max rel {worst_img:.2e}, gradients max normwise {worst_grad:.2e}")
