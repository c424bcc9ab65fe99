"""§8(f) #3 codebook consumers: oracle pinned to the reference's golden vectors
(CPU) and the CUDA drop-in against the same vectors (GPU).

Tolerances: the row ops follow NumPy's max / exp / pairwise-sum order in fp64,
so they differ from the reference only through libm exp/log ulps (rtol 1e-13);
the fp64 GEMM (decode) and BLAS-ordered dots (relevance) agree to 1e-12;
orderings (sample_tokens indices, masks) are exact.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import thinker as ot

TAGS = ("a", "b")


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_pinned_to_reference(tag):
    g = golden("thinker")
    L, E, up = g[f"{tag}_L"], g[f"{tag}_E"], g[f"{tag}_up"]
    assert np.array_equal(ot.mixture_weights(L), g[f"{tag}_w"])
    assert np.array_equal(ot.softmax_vjp(L, up), g[f"{tag}_vjp"])
    assert np.allclose(ot.decode_feature(L, E), g[f"{tag}_dec"], rtol=1e-13, atol=1e-14)
    assert np.array_equal(ot.semantic_entropy(L), g[f"{tag}_H"])
    rel = ot.contrast_scores(ot.decode_feature(L, E), g[f"{tag}_qpos"], g[f"{tag}_qneg"], 10.0)
    assert np.allclose(rel, g[f"{tag}_rel"], rtol=1e-12, atol=1e-14)
    m, fb = ot.mask_gaussians(g[f"{tag}_rel"], 0.6)
    assert np.array_equal(m, g[f"{tag}_mask"]) and fb == bool(g[f"{tag}_fallback"])
    m2, fb2 = ot.mask_gaussians(g[f"{tag}_rel"], 0.999999, 0.05)
    assert np.array_equal(m2, g[f"{tag}_mask_fb"]) and fb2 == bool(g[f"{tag}_fb2"])
    idx, H, F = ot.sample_tokens(L, E, 17)
    assert np.array_equal(idx, g[f"{tag}_tok_idx"]) and np.array_equal(H, g[f"{tag}_tok_H"])


def _stub():
    from paper_2603_09632_b200 import thinker as xt
    return xt


def test_stub_encoder_matches_reference():
    xt = _stub()
    g = golden("thinker")
    assert np.array_equal(np.stack(xt.StubTextEncoder(24).negatives()), g["neg_phrases_vecs"])
    assert np.array_equal(xt.StubTextEncoder(24).encode("a lamp"), g["hash_vec"])


def _field(xt, L):
    from paper_2603_09632_b200.core import GaussianField
    n = L.shape[0]
    return GaussianField(mu=np.zeros((n, 3)), quat=np.tile([1.0, 0, 0, 0], (n, 1)), scale=np.ones((n, 3)),
                         opacity=np.ones(n), color=np.zeros((n, 3)), logits=L)


def _cb(E):
    from paper_2603_09632_b200.core import Codebook, FeatureReservoir
    return Codebook(E=E, N=np.zeros(E.shape[0]), M=np.zeros_like(E), lam=0.96, epsilon=1e-5,
                    reservoir=FeatureReservoir(64, E.shape[1]))


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_gpu_matches_reference_golden(cuda, tag):
    xt = _stub()
    from paper_2603_09632_b200 import core
    g = golden("thinker")
    L, E, up = g[f"{tag}_L"], g[f"{tag}_E"], g[f"{tag}_up"]
    cb = _cb(E)
    assert np.allclose(core.mixture_weights(L), g[f"{tag}_w"], rtol=1e-13, atol=1e-300)
    assert np.allclose(core.softmax_vjp(L, up), g[f"{tag}_vjp"], rtol=1e-12, atol=1e-15)
    assert np.allclose(core.decode_feature(L, cb), g[f"{tag}_dec"], rtol=1e-12, atol=1e-13)
    assert np.allclose(core.decode_feature(L[5], cb), g[f"{tag}_dec1"], rtol=1e-12, atol=1e-13)
    assert np.allclose(xt.semantic_entropy(L), g[f"{tag}_H"], rtol=1e-13, atol=1e-15)
    enc = xt.StubTextEncoder(E.shape[1], region_table=E[:6])
    q = xt.TextQuery.from_prompt("region:2", enc)
    field = _field(xt, L)
    rel = xt.relevance_per_gaussian(field, cb, q)
    assert np.allclose(rel, g[f"{tag}_rel"], rtol=1e-12, atol=1e-14)
    res = xt.query_field(field, cb, q)
    assert np.array_equal(res.mask, g[f"{tag}_mask"]) and res.fallback_used == bool(g[f"{tag}_fallback"])
    m2, fb2 = xt.mask_gaussians(g[f"{tag}_rel"], 0.999999, fallback_frac=0.05)
    assert np.array_equal(m2, g[f"{tag}_mask_fb"]) and fb2 == bool(g[f"{tag}_fb2"])
    ts = xt.sample_tokens(field, cb, 17)
    assert np.array_equal(ts.indices, g[f"{tag}_tok_idx"])
    assert np.allclose(ts.entropies, g[f"{tag}_tok_H"], rtol=1e-13, atol=1e-15)
    assert np.allclose(ts.features, g[f"{tag}_tok_F"], rtol=1e-12, atol=1e-13)
    ts2 = xt.sample_tokens(field, cb, L.shape[0] + 5)
    assert np.array_equal(ts2.indices, g[f"{tag}_tok2_idx"]) and ts2.clamped
    wm = type("M", (), {"data": g[f"{tag}_wmap"]})()
    assert np.allclose(xt.relevance_per_pixel([wm], [cb], q), g[f"{tag}_relpix"], rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
def test_gpu_errors_and_edge_cases(cuda):
    xt = _stub()
    from paper_2603_09632_b200 import core
    from paper_2603_09632_b200.errors import InvalidInputError
    with pytest.raises(InvalidInputError):
        core.mixture_weights(np.array([np.nan, 0.0]))
    with pytest.raises(InvalidInputError):
        core.mixture_weights(np.array([[np.inf, 0.0], [0.0, 1.0]]))
    assert np.allclose(core.mixture_weights(np.zeros(4)), 0.25)
    w = core.mixture_weights(np.array([1000.0, 0.0, 0.0]))
    assert w[0] == 1.0 and w[1] == 0.0
    assert abs(xt.semantic_entropy(np.zeros(8)) - np.log(8)) < 1e-14
    assert xt.semantic_entropy(np.array([0.0, -1e4])) == 0.0 or xt.semantic_entropy(np.array([0.0, -1e4])) < 1e-300
    with pytest.raises(InvalidInputError):
        core.decode_feature(np.zeros(3), _cb(np.eye(4)))


@pytest.mark.gpu
def test_gpu_large_matches_oracle(cuda):
    """K=512, D=768 (the C4 codebook shape) over 50k rows; CUDA tensors in -> CUDA out."""
    import torch
    xt = _stub()
    from paper_2603_09632_b200 import core
    rng = np.random.default_rng(7)
    n, K, D = 50_000, 512, 768
    L = rng.normal(scale=2.0, size=(n, K))
    E = rng.normal(size=(K, D))
    Ld = torch.from_numpy(L).cuda()
    H = xt.semantic_entropy(Ld).cpu().numpy()
    assert np.allclose(H, ot.semantic_entropy(L), rtol=1e-13, atol=1e-15)
    cb = _cb(E).to_device()
    idx = rng.integers(0, n, 300)
    F = core.decode_feature(Ld[torch.from_numpy(idx).cuda()], cb).cpu().numpy()
    assert np.allclose(F, ot.decode_feature(L[idx], E), rtol=1e-11, atol=1e-12)
    ts = xt.sample_tokens(type("F", (), {"logits": Ld, "__len__": lambda self: n})(), cb, 1000)
    o, Hs, _ = ot.sample_tokens(L, E, 1000)
    assert np.array_equal(ts.indices.cpu().numpy(), o)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["normal", "ties", "all_equal", "signed_zero", "wide_range"])
@pytest.mark.parametrize("M", [1, 37, 2500])
def test_desc_top_m_matches_stable_argsort(cuda, case, M):
    """xgs_desc_top_m (bucket select + stable sort of the candidates) ==
    np.argsort(-v, kind="stable")[:M], ties to the lower index."""
    import torch
    from paper_2603_09632_b200 import thinker
    rng = np.random.default_rng(M)
    n = 20_000
    if case == "normal":
        v = rng.normal(size=n)
    elif case == "ties":
        v = rng.integers(0, 7, n).astype(np.float64)
    elif case == "all_equal":
        v = np.full(n, 0.25)
    elif case == "signed_zero":
        v = np.where(rng.random(n) < 0.5, 0.0, -0.0) * (rng.random(n) < 0.9) + (rng.random(n) < 0.001)
    else:
        v = rng.normal(size=n) * 10.0 ** rng.integers(-30, 30, n)
    got = thinker._desc_top_m(torch.from_numpy(v).cuda(), M).cpu().numpy()
    assert np.array_equal(got, np.argsort(-v, kind="stable")[:M])


@pytest.mark.gpu
@pytest.mark.parametrize("n,kr,m", [(1, 5, 3), (33, 17, 385), (1000, 512, 768), (257, 100, 1000)])
@pytest.mark.parametrize("layout", ["softmax", "plain", "a_t", "b_t"])
def test_gemm_f64_dmma_shapes(cuda, n, kr, m, layout):
    """xgs_gemm_f64 (DMMA fp64, softmax prologue / strided operands / contrast
    epilogue) against NumPy fp64 at tile-edge shapes."""
    import torch
    from paper_2603_09632_b200 import core
    rng = np.random.default_rng(n + kr + m)
    A = rng.normal(scale=2.0, size=(n, kr))
    B = rng.normal(size=(kr, m))
    if layout == "softmax":
        W = np.exp(A - A.max(axis=1, keepdims=True))
        W /= W.sum(axis=1, keepdims=True)
        ref = W @ B
        got = core.gemm_f64(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), softmax=True)
    elif layout == "plain":
        ref = A @ B
        got = core.gemm_f64(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    elif layout == "a_t":
        ref = A @ B
        got = core.gemm_f64(torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), torch.from_numpy(B).cuda(),
                            a_transposed=True)
    else:
        ref = A @ B
        got = core.gemm_f64(torch.from_numpy(A).cuda(), torch.from_numpy(np.ascontiguousarray(B.T)).cuda(),
                            b_transposed=True)
    np.testing.assert_allclose(got.cpu().numpy(), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    if layout == "softmax" and m >= 2:
        Q = rng.normal(size=(3, m))
        Q /= np.linalg.norm(Q, axis=1, keepdims=True)
        f = ref / (np.linalg.norm(ref, axis=1, keepdims=True) + 1e-8)
        pos = f @ Q[0]
        sc = np.ones(n)
        for q in Q[1:]:
            sc = np.minimum(sc, 1.0 / (1.0 + np.exp(-(10.0 * (pos - f @ q)))))
        _, s2 = core.gemm_f64(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), softmax=True,
                              query=torch.from_numpy(Q).cuda(), tau=10.0, eps=1e-8, want_c=False)
        np.testing.assert_allclose(s2.cpu().numpy(), sc, rtol=1e-12, atol=1e-14)
