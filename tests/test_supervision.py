"""Grid-sampled supervision targets against the reference's
golden vectors (tests/golden/supervision.npz) and the oracle restatement.
Targets / padding / masks / cotangents bit-exact; the scalar loss (a mean over
cells, summed in a different order) within 1e-12 relative."""

import numpy as np
import pytest

from conftest import golden
from oracle import supervision as osup


def test_oracle_matches_reference_golden():
    g = golden("supervision")
    H, W = 37, 53
    for i, (s, oh, ow) in enumerate(g["cases"]):
        Gc, _ = osup.target_continuous(g["P"], H, W, s, oh, ow)
        assert np.array_equal(Gc, g[f"cont_G_{i}"])
        Gd, Vd = osup.target_discrete(g["S"], g["Phi"], H, W, s, oh, ow)
        assert np.array_equal(Gd, g[f"disc_G_{i}"]) and np.array_equal(Vd, g[f"disc_V_{i}"])
        Gp, Vp = osup.pad(Gd, Vd, H, W, s)
        assert np.array_equal(Gp, g[f"pad_G_{i}"]) and np.array_equal(Vp, g[f"pad_V_{i}"])
        loss, cot = osup.semantic_loss(g[f"pred_{i}"], Gd, Vd, 0.7)
        assert loss == float(g[f"loss_{i}"]) and np.array_equal(cot, g[f"cot_{i}"])
    assert [osup.next_offset(k, 4, 3) for k in range(40)] == [tuple(o) for o in g["offsets"]]


def test_host_lattice_api_matches_reference_golden():
    from paper_2603_09632_b200 import supervision as sup
    g = golden("supervision")
    assert [sup.next_offset(k, 4, 3) for k in range(40)] == [tuple(o) for o in g["offsets"]]
    assert [sup.next_offset(k, 1, 3) for k in range(3)] == [tuple(o) for o in g["offsets_s1"]]
    assert sup.grid_resolution(480, 4, 0) == 120 and sup.grid_resolution(3, 5, 4) == 0
    with pytest.raises(sup.InvalidInputError):
        sup.grid_resolution(10, 3, 3)
    spec = sup.GridSpec(5, 6, 2, 1, 0)
    assert sup.sample_coordinates(spec).tolist() == [[1, 0], [1, 2], [1, 4], [3, 0], [3, 2], [3, 4]]


@pytest.mark.gpu
def test_gpu_targets_match_reference_golden(cuda):
    from paper_2603_09632_b200 import supervision as sup
    g = golden("supervision")
    H, W = 37, 53
    src = sup.ContinuousFeatureSource(g["P"])
    ann = sup.RegionAnnotation(g["S"], g["Phi"])
    for i, (s, oh, ow) in enumerate(g["cases"]):
        spec = sup.GridSpec(H, W, int(s), int(oh), int(ow))
        tc = sup.build_target_continuous(src, spec)
        assert np.array_equal(tc.G_star, g[f"cont_G_{i}"]) and (tc.V == 1).all()
        td = sup.build_target_discrete(ann, spec)
        assert np.array_equal(td.G_star, g[f"disc_G_{i}"]) and np.array_equal(td.V, g[f"disc_V_{i}"])
        pt = sup.pad_target(td, spec)
        assert np.array_equal(pt.G_star, g[f"pad_G_{i}"]) and np.array_equal(pt.V, g[f"pad_V_{i}"])
        loss, cot = sup.masked_semantic_loss(g[f"pred_{i}"], td, lambda_sem=0.7)
        np.testing.assert_allclose(loss, float(g[f"loss_{i}"]), rtol=1e-12)
        assert np.array_equal(cot, g[f"cot_{i}"])


@pytest.mark.gpu
def test_gpu_prefetch_equals_per_offset_targets(cuda):
    from paper_2603_09632_b200 import supervision as sup
    rng = np.random.default_rng(3)
    H, W, s = 60, 80, 4
    P = rng.normal(size=(9, 4, 5)).astype(np.float32)
    src = sup.ContinuousFeatureSource(P)
    G, V = sup.prefetch_targets(src, H, W, s, range(16), rng_seed=2)
    for k in range(16):
        oh, ow = sup.next_offset(k, s, 2)
        Gr, Vr = osup.target_continuous(P.astype(np.float64), H, W, s, oh, ow)
        Gp, Vp = osup.pad(Gr, Vr, H, W, s)
        assert np.array_equal(G[k].cpu().numpy(), Gp) and np.array_equal(V[k].cpu().numpy(), Vp), k
    S = rng.integers(-1, 3, (H, W))
    S[0, 0] = 7
    with pytest.raises(sup.CorruptAnnotationError):
        sup.build_target_discrete(sup.RegionAnnotation(S, rng.normal(size=(3, 4))), sup.GridSpec(H, W, 2, 0, 0))
