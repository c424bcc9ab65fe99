"""The reference's OWN test module for the hot path (semsplat pkg/tests/test_vq.py,
unmodified) run against the B200 path: paper_2603_09632_b200.reference_shim is
installed over the pip-installed reference (baseline/_ref, see
tools/install_reference.sh) before the module is imported, so every
``semsplat.vq`` call in it -- with the reference's own Codebook /
FeatureReservoir objects and error classes -- runs on libxgs.

Skipped when baseline/_ref (git-ignored; it travels to the GPU box with the
working tree) was not installed."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "semsplat_tests")


def _run(test_file, extra=()):
    if not os.path.isfile(os.path.join(SUITE, test_file)):
        pytest.skip("reference not installed under baseline/_ref (tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests"), ROOT, env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "_ref_shim_plugin", "-p", "no:cacheprovider",
           "--rootdir", SUITE, "-o", "addopts=", os.path.join(SUITE, test_file), *extra]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200, cwd=SUITE)
    return r


def test_reference_test_vq_passes_through_shim(cuda):
    r = _run("test_vq.py")
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "24 passed" in r.stdout, r.stdout[-2000:]
    import re
    m = re.search(r"B200 shim installed over semsplat: 13 functions; libxgs kernel launches: (\d+)", r.stdout)
    assert m and int(m.group(1)) > 1000, r.stdout[-2000:]     # the suite ran on libxgs, not NumPy


def test_shim_routes_to_native(cuda):
    """The installed functions are the adapters (not the NumPy reference), they
    return the reference's types and raise the reference's errors."""
    if not os.path.isdir(os.path.join(REF, "semsplat")):
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import numpy as np
        import semsplat.core as rc
        import semsplat.errors as re_
        import semsplat.vq as rv

        from paper_2603_09632_b200 import _native, reference_shim
        reference_shim.install()
        try:
            assert getattr(rv.online_step, "__b200__", False)
            rng = np.random.default_rng(0)
            E = rng.normal(size=(8, 5))
            cb = rc.Codebook(E=E, N=np.zeros(8), M=np.zeros((8, 5)), lam=0.9, epsilon=1e-5,
                             reservoir=rc.FeatureReservoir(16, 5))
            n0 = _native.launch_count()
            cb2, res = rv.online_step(cb, rng.normal(size=(40, 5)), rv.VqConfig(K=8, lam=0.9), rng)
            assert _native.launch_count() > n0          # libxgs kernels ran
            assert isinstance(cb2, rc.Codebook) and isinstance(res, rv.ReviveResult)
            assert cb2.reservoir is cb.reservoir and len(cb.reservoir) == 16
            with pytest.raises(re_.InvalidInputError):
                rv.assign(np.zeros(4), cb2)
            with pytest.raises(re_.InvalidStateError):
                rv.assign_batch(np.zeros((1, 0)), rc.Codebook(E=np.zeros((0, 0)), N=np.zeros(0),
                                                              M=np.zeros((0, 0)), lam=0.5, epsilon=1e-5))
        finally:
            reference_shim.uninstall()
    finally:
        sys.path.remove(REF)


def test_shim_slam_matches_reference(cuda):
    """backproject / densify_and_prune through the shim on the reference's own
    types (a scene, trajectory and frames from semsplat.world) give the same
    splats as the reference's NumPy functions on the same inputs."""
    if not os.path.isdir(os.path.join(REF, "semsplat")):
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import numpy as np
        import semsplat.core as rc
        import semsplat.slam as rs
        import semsplat.world as rw

        from paper_2603_09632_b200 import _native, reference_shim
        recipe = rw.standard_recipe(height=48, width=64, n_gaussians=90)
        field, labels, phi = rw.generate_scene(recipe)
        poses = rw.generate_trajectory(recipe)
        frames = rw.render_ground_truth(field, labels, phi, poses[:12:4], recipe.intrinsics())
        cfg = rs.SlamConfig()
        reference_shim.install()
        try:
            ref_bp, ref_dp = rs.backproject.__wrapped_reference__, rs.densify_and_prune.__wrapped_reference__
            intr = rs.frame_intrinsics(frames[0], cfg)
            for (u, v, d) in ((0.0, 0.0, 1.0), (17.5, 30.25, 2.75), (63.0, 47.0, 0.4)):
                assert np.array_equal(rs.backproject(poses[4], intr, u, v, d), ref_bp(poses[4], intr, u, v, d))
            keep = np.random.default_rng(3).random(len(field)) < 0.5      # leave holes to fill
            part = rc.GaussianField(mu=field.mu[keep], quat=field.quat[keep], scale=field.scale[keep],
                                    opacity=np.where(np.arange(keep.sum()) % 9 == 0, 0.004, field.opacity[keep]),
                                    color=field.color[keep], logits=np.zeros((int(keep.sum()), 4)))
            empty = rc.GaussianField(mu=np.zeros((0, 3)), quat=np.zeros((0, 4)), scale=np.zeros((0, 3)),
                                     opacity=np.zeros(0), color=np.zeros((0, 3)), logits=np.zeros((0, 4)))
            for fr in frames:
                win = rs.KeyframeWindow(3)
                win.insert(fr, fr.pose)
                for start in (part, empty):
                    n0 = _native.launch_count()
                    got = rs.densify_and_prune(start, win, cfg, K=4)
                    assert _native.launch_count() > n0
                    ref = ref_dp(start, win, cfg, K=4)
                    assert isinstance(got, rc.GaussianField) and len(got) == len(ref), fr.frame_id
                    for name in ("mu", "quat", "scale", "opacity", "color", "logits"):
                        assert np.array_equal(getattr(got, name), getattr(ref, name)), (fr.frame_id, name)
                    assert got.generation == ref.generation
        finally:
            reference_shim.uninstall()
    finally:
        sys.path.remove(REF)
