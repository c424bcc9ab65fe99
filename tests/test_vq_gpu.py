"""GPU parity of the VQ drop-in against the reference's golden vectors, the
restated reference KATs (pkg/tests/test_vq.py) and the CPU oracle.

Tolerances: codes / counts / sums / E / N / M are compared bit-exactly
(array_equal); softmax probabilities (libm exp) with rtol 1e-13.
"""

import itertools

import numpy as np
import pytest

from conftest import golden
from oracle import native as on
from oracle import vq as ov

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xv(cuda):
    import paper_2603_09632_b200 as xv
    return xv


def make_cb(xv, E, lam=0.96, eps=1e-5, cap=64):
    E = np.asarray(E, dtype=float)
    return xv.Codebook(E=E, N=np.zeros(E.shape[0]), M=np.zeros_like(E), lam=lam, epsilon=eps,
                       reservoir=xv.FeatureReservoir(cap, E.shape[1]))


def mixture(rng, n, D, centres, sigma, dtype=np.float32):
    C = rng.normal(size=(centres, D))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    x = C[rng.integers(0, centres, n)] + sigma * rng.normal(size=(n, D))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x.astype(dtype)


# ------------------------------------------------------------ golden vectors

def test_squared_distances_golden(xv):
    g = golden("sqdist")
    for D in (1, 3, 7, 8, 9, 17, 100, 128, 129, 255, 512, 768, 1152):
        got = xv.squared_distances(g[f"x_{D}"], make_cb(xv, g[f"E_{D}"]))
        assert np.array_equal(got, g[f"d_{D}"]), D


def test_assign_golden(xv):
    g = golden("assign")
    for case in ("c1", "c2", "tie", "tie2"):
        cb = make_cb(xv, g[f"{case}_E"].astype(np.float64))
        assert np.array_equal(xv.assign_batch(g[f"{case}_x"], cb), g[f"{case}_codes"]), case


def test_accumulate_ema_golden(xv):
    g = golden("accumulate")
    cb = make_cb(xv, g["E"], lam=0.99)
    st = xv.accumulate(g["x"], cb)
    assert np.array_equal(st.counts, g["counts"]) and np.array_equal(st.sums, g["sums"])
    cb.N[:] = g["N0"]
    cb.M[:] = g["M0"]
    e = xv.ema_step(cb, st)
    assert np.array_equal(e.N, g["N1"]) and np.array_equal(e.M, g["M1"]) and np.array_equal(e.E, g["E1"])


def test_online_step_golden_confidence_path(xv):
    g = golden("online")
    cfg = xv.VqConfig(K=4, lam=0.8, gamma=0.5, tau_warm=0.7, delta_dead=1e-2)
    cb = make_cb(xv, g["a_E0"], lam=0.8, cap=128)
    rng = np.random.default_rng(7)
    for i, b in enumerate(g["a_batches"]):
        cb, res = xv.online_step(cb, b, cfg, rng)
        assert np.array_equal(cb.E, g["a_E"][i]) and np.array_equal(cb.N, g["a_N"][i]), i
        assert np.array_equal(cb.M, g["a_M"][i]) and len(res.revived) == g["a_nrev"][i]


def test_online_step_golden_baseline_path(xv):
    g = golden("online")
    K = 64
    cfg = xv.VqConfig(K=K, lam=0.99, gamma=0.5 / K, delta_dead=1e-3)
    for device in (False, True):
        cb = make_cb(xv, g["b_E0"], lam=0.99, cap=300)
        if device:
            cb = cb.to_device()
        rng = np.random.default_rng(12)
        x = g["b_x"]
        for i in range(8):
            b = x[i * 256:(i + 1) * 256]
            if device:
                import torch
                b = torch.from_numpy(b).cuda()
            cb, res = xv.online_step(cb, b, cfg, rng)
            c = cb.to_numpy()
            assert np.array_equal(c.E, g["b_E"][i]) and np.array_equal(c.N, g["b_N"][i]), (device, i)
            assert len(res.revived) == g["b_nrev"][i]


def test_confidence_golden(xv):
    g = golden("online")
    cb = make_cb(xv, g["c_E"])
    p = xv.confidence_scores(g["c_x"], cb, 0.7)
    np.testing.assert_allclose(p, g["c_p"], rtol=1e-13, atol=0)
    assert np.array_equal(xv.confidence_mask(g["c_x"], cb, xv.VqConfig(K=7, gamma=0.4)), g["c_mask"])


def test_warm_start_and_seeding_golden(xv):
    g = golden("online")
    seeds = xv.seed_from_samples(g["d_buf"], 4)
    assert np.array_equal(seeds, g["d_seeds"])
    ws = xv.warm_start(g["d_buf"], make_cb(xv, seeds), xv.VqConfig(K=4, gamma=0.3))
    assert not ws.degenerate and ws.used == int(g["d_used"])
    assert np.array_equal(ws.codebook.E, g["d_E"]) and np.array_equal(ws.codebook.N, g["d_N"])


@pytest.mark.parametrize("case", ["mixture_f32", "odd_d_f64", "cycling", "single_row", "nan_row", "ties",
                                  "bf16", "k_le_1"])
@pytest.mark.parametrize("coop", ["1", "0"])
def test_seed_from_samples_matches_oracle(xv, case, coop, monkeypatch):
    """Device farthest-point seeding (xgs_vq_seed_farthest) vs the oracle
    restatement of vq.py:126-147, bit-exact: argmax ties to the lower index,
    cycling once the maximum is 0, NaN rows first (np.argmax / np.minimum)."""
    import torch
    rng = np.random.default_rng(77)
    K = 24
    if case == "mixture_f32":
        buf, K = mixture(rng, 3000, 512, 40, 0.05), 64
    elif case == "odd_d_f64":
        buf = rng.normal(size=(777, 301))
    elif case == "cycling":      # 3 distinct rows, K > 3: seeds cycle through the buffer
        buf = np.repeat(rng.normal(size=(3, 16)), 4, axis=0)
    elif case == "single_row":
        buf = rng.normal(size=(1, 8))
    elif case == "nan_row":
        buf = rng.normal(size=(50, 8))
        buf[17, 3] = np.nan
    elif case == "ties":         # integer lattice: many equal distances
        buf = rng.integers(0, 3, size=(200, 4)).astype(np.float64)
    elif case == "bf16":
        buf = torch.from_numpy(mixture(rng, 500, 128, 8, 0.1)).to(torch.bfloat16).cuda()
    else:
        buf, K = rng.normal(size=(10, 5)), 0
    monkeypatch.setenv("XGS_SEED_NO_COOP", "0" if coop == "1" else "1")   # cooperative or per-launch path
    want = ov.seed_from_samples(buf.float().cpu().numpy() if torch.is_tensor(buf) else buf, K)
    got = xv.seed_from_samples(buf, K)
    got = got.cpu().numpy() if torch.is_tensor(got) else got
    assert got.shape == want.shape
    assert np.array_equal(got, want, equal_nan=True)


# ------------------------------------------- restated reference KATs (test_vq.py)

def test_kat_assign(xv):
    rng = np.random.default_rng(21)
    cb = make_cb(xv, rng.normal(size=(5, 3)))
    assert xv.assign(cb.E[3], cb) == 3                                   # :30-32
    assert xv.assign(np.array([1.0]), make_cb(xv, [[0.0], [2.0]])) == 0  # :34-36
    cb = make_cb(xv, rng.normal(size=(17, 6)))                          # :38-44
    xs = rng.normal(size=(200, 6))
    got = xv.assign_batch(xs, cb)
    for n in range(200):
        assert got[n] == int(np.argmin([np.linalg.norm(xs[n] - cb.E[k]) for k in range(17)]))
    with pytest.raises(xv.InvalidInputError):                           # :46-49
        xv.assign(np.zeros(4), make_cb(xv, np.eye(3)))
    with pytest.raises(xv.InvalidStateError):
        xv.assign_batch(np.zeros((2, 3)), make_cb(xv, np.zeros((0, 3))))


def test_kat_accumulate(xv):
    rng = np.random.default_rng(22)
    cb = make_cb(xv, np.eye(4))                                          # :53-60
    st = xv.accumulate(np.tile(cb.E[2], (5, 1)), cb)
    assert st.counts[2] == 5 and np.allclose(st.sums[2], 5 * cb.E[2]) and st.counts.sum() == 5
    assert not st.sums[[0, 1, 3]].any()
    cb = make_cb(xv, rng.normal(size=(6, 3)))                            # :67-78
    batch = rng.normal(size=(40, 3))
    st = xv.accumulate(batch, cb)
    counts, sums = np.zeros(6), np.zeros((6, 3))
    for x in batch:
        k = xv.assign(x, cb)
        counts[k] += 1
        sums[k] += x
    assert np.array_equal(st.counts, counts) and np.array_equal(st.sums, sums)
    with pytest.raises(xv.InvalidInputError):
        xv.accumulate(np.zeros((0, 3)), cb)


def test_kat_ema(xv):
    rng = np.random.default_rng(23)
    cb = make_cb(xv, rng.normal(size=(3, 2)), lam=0.0)                   # :88-94
    st = xv.accumulate(rng.normal(size=(10, 2)), cb)
    out = xv.ema_step(cb, st)
    assert np.array_equal(out.N, st.counts) and np.array_equal(out.M, st.sums)
    cb = make_cb(xv, rng.normal(size=(4, 2)), lam=0.96)                  # :103-114
    cb.N[:] = np.array([1.0, 2.0, 0.5, 7.0])
    ref = cb.N.copy()
    zero = xv.VqBatchStats(counts=np.zeros(4), sums=np.zeros((4, 2)))
    for _ in range(30):
        cb = xv.ema_step(cb, zero)
        ref = 0.96 * ref
        assert np.array_equal(cb.N, ref)
    cb = make_cb(xv, rng.normal(size=(5, 3)))                            # :116-122
    r2 = np.random.default_rng(0)
    for _ in range(10):
        cb, _ = xv.online_step(cb, r2.normal(size=(20, 3)), xv.VqConfig(K=5), r2)
        assert np.allclose(cb.E, cb.M / (cb.N + cb.epsilon)[:, None], atol=1e-12)


def test_kat_streaming_converges_to_kmeans(xv):  # test_vq.py:133-165
    rng = np.random.default_rng(77)
    centers = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [0.0, 0, 1]])
    stream = lambda n: centers[rng.choice(4, size=n)] + rng.normal(0, 0.01, (n, 3))
    cfg = xv.VqConfig(K=4, lam=0.96)
    first = stream(64)
    pooled = [first]
    cb = make_cb(xv, xv.seed_from_samples(first, 4), lam=0.96)
    cb = xv.warm_start(first, cb, cfg).codebook
    for _ in range(200):
        b = stream(64)
        pooled.append(b)
        cb, _ = xv.online_step(cb, b, cfg, rng)
    data = np.concatenate(pooled)
    km = [data[0]]
    for _ in range(3):
        d = np.min([np.linalg.norm(data - c, axis=1) for c in km], axis=0)
        km.append(data[int(d.argmax())])
    km = np.stack(km)
    for _ in range(50):
        a = ((data[:, None] - km[None]) ** 2).sum(axis=2).argmin(axis=1)
        km = np.stack([data[a == k].mean(axis=0) for k in range(4)])
    best = min(np.abs(cb.E[list(p)] - km).max() for p in itertools.permutations(range(4)))
    assert best < 0.05


def test_kat_dead_codes(xv):
    rng = np.random.default_rng(24)
    cb = make_cb(xv, rng.normal(size=(2, 2)))                            # :218-232
    cb.N[:] = [1.0, 0.0]
    v = np.array([3.0, -1.0])
    cb.reservoir.extend(v[None])
    res = xv.revive_dead_codes(cb, xv.VqConfig(K=2), np.random.default_rng(0))
    assert res.revived == [1]
    assert np.allclose(res.codebook.E[1], v / (1 + 2e-5)) and np.allclose(res.codebook.N[1], 1 + 1e-5)
    cb = make_cb(xv, rng.normal(size=(2, 2)))                            # :234-238
    cb.N[:] = [1.0, 0.0]
    res = xv.revive_dead_codes(cb, xv.VqConfig(K=2), np.random.default_rng(0))
    assert res.skipped and res.revived == []


# ------------------------------------------------------ oracle parity at scale

@pytest.mark.parametrize("n,K,D", [(20000, 1024, 512), (4096, 256, 512), (3000, 512, 768),
                                   (1500, 4096, 1152), (777, 37, 3), (513, 300, 129)])
def test_assign_matches_oracle(xv, n, K, D):
    rng = np.random.default_rng(n + K + D)
    x = mixture(rng, n, D, max(4, K), 0.05)
    E = mixture(rng, K, D, max(4, K), 0.05).astype(np.float64)
    cb = make_cb(xv, E)
    got, (nr, nf) = xv.vq.assign_batch_stats(x, cb)
    ref = on.assign(x, E, threads=8)
    assert np.array_equal(got, ref)
    print(f"n={n} K={K} D={D}: rerank {nr} fallback {nf}")


@pytest.mark.parametrize("D", [1152, 100])
def test_assign_bf16_rows(xv, D):
    """bf16 rows: D=1152 takes the 16-byte vector prep path, D=100 the scalar one."""
    import torch
    rng = np.random.default_rng(5)
    x = torch.from_numpy(mixture(rng, 5000, D, 512, 0.05)).to(torch.bfloat16).cuda()
    E = mixture(rng, 512, D, 512, 0.05).astype(np.float64)
    cb = make_cb(xv, E).to_device()
    got = xv.assign_batch(x, cb).cpu().numpy()
    ref = on.assign(x.cpu().view(torch.int16).numpy().view(np.uint16), E, threads=8, bf16=True)
    assert np.array_equal(got, ref)
    st = xv.accumulate(x, cb)
    c, s = on.accumulate(x.cpu().view(torch.int16).numpy().view(np.uint16), ref, 512, bf16=True)
    assert np.array_equal(st.counts.cpu().numpy(), c) and np.array_equal(st.sums.cpu().numpy(), s)


def test_duplicate_codewords_and_exact_hits(xv):
    rng = np.random.default_rng(9)
    E = rng.normal(size=(64, 96))
    E[10:30] = E[5]                      # 21 identical codewords -> candidate overflow
    x = np.concatenate([E[[5, 10, 40]], rng.normal(size=(300, 96)), np.tile(E[5], (40, 1)) + 1e-9])
    cb = make_cb(xv, E)
    got, (nr, nf) = xv.vq.assign_batch_stats(x, cb)
    assert np.array_equal(got, on.assign(x, E))
    assert got[0] == 5 and got[1] == 5 and nf > 0


def test_online_step_device_matches_oracle(xv):
    import torch
    rng = np.random.default_rng(31)
    n, K, D = 8192, 256, 512
    x = mixture(rng, n * 4, D, 64, 0.1)
    E0 = x[rng.choice(x.shape[0], K, replace=False)].astype(np.float64)
    cfg = xv.VqConfig(K=K, lam=0.99, gamma=0.5 / K, delta_dead=1e-3)
    cb = make_cb(xv, E0, lam=0.99, cap=4096).to_device()
    oc = ov.OracleCodebook(E0, np.zeros(K), np.zeros((K, D)), 0.99, 1e-5, ov.OracleReservoir(4096, D))
    r1, r2 = np.random.default_rng(4), np.random.default_rng(4)
    xd = torch.from_numpy(x).cuda()
    for i in range(4):
        b = x[i * n:(i + 1) * n]
        cb, res = xv.online_step(cb, xd[i * n:(i + 1) * n], cfg, r1)
        # oracle step with the fast C assign (bit-identical to the NumPy restatement)
        oc.reservoir.extend(b)
        codes = on.assign(b, oc.E, threads=8)
        counts, sums = on.accumulate(b, codes, K)
        oc = ov.ema_step(oc, counts, sums)
        oc, rev, _ = ov.revive_dead_codes(oc, 1e-3, r2)
        c = cb.to_numpy()
        assert np.array_equal(c.N, oc.N) and np.array_equal(c.M, oc.M) and np.array_equal(c.E, oc.E), i
        assert res.revived == rev
    assert np.array_equal(cb.reservoir.as_array(), oc.reservoir.buf)


@pytest.mark.parametrize("n,K,D,dtype", [(700_000, 256, 64, "f32"), (400_000, 512, 96, "bf16"),
                                         (300_000, 128, 40, "f64")])
def test_pipelined_assign_accumulate(xv, n, K, D, dtype):
    """xgs_vq_assign_accumulate (row-chunk pipeline, >= 2 chunks at these n)
    is bit-identical to assign + accumulate and to the C oracle."""
    import torch
    from paper_2603_09632_b200 import vq as xvq
    rng = np.random.default_rng(n + K)
    x = mixture(rng, n, D, K, 0.05)
    E = mixture(rng, K, D, K, 0.05).astype(np.float64)
    if dtype == "bf16":
        xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
        xh = xt.cpu().view(torch.int16).numpy().view(np.uint16)
    else:
        xt = torch.from_numpy(x.astype(np.float64) if dtype == "f64" else x).cuda()
        xh = xt.cpu().numpy()
    Et = torch.from_numpy(E).cuda()
    r, dt, nn, d, ldx = xvq._rows(xt)
    codes, counts, sums = xvq._assign_accumulate_dev(r, dt, nn, d, ldx, Et, K)
    codes2 = xvq._assign_dev(r, dt, nn, d, ldx, Et, K)
    counts2, sums2 = xvq._accumulate_dev(r, dt, nn, d, ldx, codes2, None, K)
    assert torch.equal(codes, codes2)
    assert torch.equal(counts, counts2) and torch.equal(sums, sums2)
    ref = on.assign(xh, E, threads=8, bf16=dtype == "bf16")
    assert np.array_equal(codes.cpu().numpy(), ref)
    c, sm = on.accumulate(xh, ref, K, bf16=dtype == "bf16")
    assert np.array_equal(counts.cpu().numpy(), c) and np.array_equal(sums.cpu().numpy(), sm)


@pytest.mark.parametrize("n,K,D,skew", [(50_000, 1024, 64, False), (50_000, 1024, 64, True),
                                        (20_000, 8192, 16, False), (30_000, 50_000, 8, False), (1025, 7, 33, True)])
def test_accumulate_counting_sort_paths(xv, n, K, D, skew):
    """accumulate over given codes + confidence mask at n > 1024: the
    block-per-tile counting sort (K <= 40960; 8 warps per tile, fewer at
    K = 8192), the per-warp-tile fallback (K = 50000), skewed code counts
    (one code holds half the rows: the longest chain) -- bit-identical to
    bincount + np.add.at over the masked rows."""
    import torch
    from paper_2603_09632_b200 import vq as xvq
    rng = np.random.default_rng(n + K)
    x = rng.normal(size=(n, D)).astype(np.float32)
    codes = rng.integers(0, K, n)
    if skew:
        codes[rng.random(n) < 0.5] = K // 2
    mask = rng.random(n) < 0.9
    xt = torch.from_numpy(x).cuda()
    r, dt, nn, d, ldx = xvq._rows(xt)
    counts, sums = xvq._accumulate_dev(r, dt, nn, d, ldx, torch.from_numpy(codes).cuda(),
                                       torch.from_numpy(mask).cuda(), K)
    c, sm = on.accumulate(x[mask], codes[mask], K)
    assert np.array_equal(counts.cpu().numpy(), c) and np.array_equal(sums.cpu().numpy(), sm)


def test_assign_edge_cases(xv):
    rng = np.random.default_rng(11)
    # single row, single code, D = 1
    cb = make_cb(xv, [[0.5]])
    assert xv.assign_batch(np.array([[3.0]]), cb).tolist() == [0]
    # all-identical codebook (Codebook.zeros): every row ties -> lowest index 0 (overflow path)
    cb = xv.Codebook.zeros(40, 16)
    x = rng.normal(size=(300, 16))
    codes, (nr, nf) = xv.vq.assign_batch_stats(x, cb)
    assert (codes == 0).all() and nf == 300
    # extreme magnitudes: power-of-two scaling keeps the fp16 screen exact enough
    E = rng.normal(size=(50, 24))
    for scale in (1e-30, 1e-8, 1.0, 1e8, 1e30):
        xs = rng.normal(size=(200, 24)) * scale
        cbs = make_cb(xv, E * scale)
        assert np.array_equal(xv.assign_batch(xs, cbs), on.assign(xs, E * scale)), scale
    # zero rows and rows equal to codewords
    xs = np.concatenate([np.zeros((3, 24)), E[[7, 7, 49]]])
    assert np.array_equal(xv.assign_batch(xs, make_cb(xv, E)), on.assign(xs, E))


def test_float64_and_strided_inputs(xv):
    import torch
    rng = np.random.default_rng(12)
    E = rng.normal(size=(300, 40))
    x = rng.normal(size=(1000, 80))[:, ::2]          # non-contiguous float64 view
    assert np.array_equal(xv.assign_batch(x, make_cb(xv, E)), on.assign(np.ascontiguousarray(x), E))
    xt = torch.from_numpy(rng.normal(size=(1000, 48)).astype(np.float32)).cuda()[:, :40]   # ldx = 48
    got = xv.assign_batch(xt, make_cb(xv, E).to_device()).cpu().numpy()
    assert np.array_equal(got, on.assign(xt.cpu().numpy(), E))
    st = xv.accumulate(xt, make_cb(xv, E).to_device())
    c, s = on.accumulate(xt.cpu().numpy(), got, 300)
    assert np.array_equal(st.counts.cpu().numpy(), c) and np.array_equal(st.sums.cpu().numpy(), s)


def test_pinned_host_batch_streams_bit_identical(xv):
    """DataParallelVQ on a pinned host batch (rows streamed H2D chunk by chunk
    inside the pipelined call) == the same steps on the device batch."""
    import torch
    from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
    rng = np.random.default_rng(77)
    n, K, D = 400_000, 256, 64
    x = mixture(rng, n, D, K, 0.05)
    E0 = torch.from_numpy(mixture(rng, K, D, K, 0.05).astype(np.float64)).cuda()
    cfg = xv.VqConfig(K=K, lam=0.99, gamma=0.5 / K, delta_dead=1e-3, reservoir_capacity=512)
    runs = []
    for src in (torch.from_numpy(x).cuda(), torch.from_numpy(x).pin_memory()):
        st = (E0.clone(), torch.zeros(K, dtype=torch.float64, device="cuda"),
              torch.zeros(K, D, dtype=torch.float64, device="cuda"))
        vq = DataParallelVQ(st, cfg, np.random.default_rng(3), CudaBackend(K, D, 0.99, 1e-5))
        for _ in range(3):
            vq.step(src, [n])
        runs.append([s.cpu().numpy() for s in vq.state] + [vq.ring.cpu().numpy()])
    for a, b in zip(*runs):
        assert np.array_equal(a, b)


def test_confidence_mask_rows_at_gamma(xv):
    """Rows whose max softmax lies at / within an ulp of gamma (SURVEY §7 hard
    part 5): the kernel marks them undecided and they are decided with the
    reference's own NumPy expression -- the mask equals the reference's."""
    rng = np.random.default_rng(17)
    E = rng.normal(size=(40, 24))
    x = rng.normal(size=(300, 24))
    x[0] = 0.5 * (E[3] + E[7])          # exactly equidistant from two codes
    cb = make_cb(xv, E)
    sq = ((x[:, None, :] - E[None, :, :]) ** 2).sum(axis=2)
    lg = -np.sqrt(sq) / 0.7
    lg -= lg.max(axis=1, keepdims=True)
    e = np.exp(lg)
    pmax = (e / e.sum(axis=1, keepdims=True)).max(axis=1)
    for gamma in (pmax[0], pmax[5], np.nextafter(pmax[5], 1.0), np.nextafter(pmax[9], 0.0), 0.3):
        cfg = xv.VqConfig(K=40, tau_warm=0.7, gamma=float(gamma))
        got = xv.confidence_mask(x, cb, cfg)
        assert np.array_equal(got, pmax >= gamma), gamma


@pytest.mark.parametrize("K", [256, 4096])
def test_assign_with_device_row_count(xv, K):
    """xgs_vq_assign_dev: rows [0, min(*n_dev, n)) get the codes xgs_vq_assign
    gives them; rows past the count are left untouched."""
    import torch

    from paper_2603_09632_b200 import _native as nat
    rng = np.random.default_rng(77)
    n, D = 3000, 96
    x = torch.from_numpy(rng.normal(size=(n, D)).astype(np.float32)).cuda()
    E = torch.from_numpy(rng.normal(size=(K, D))).cuda()
    L = nat.lib()
    ws = nat.workspace("t_assign_dev", L.xgs_vq_assign_workspace(n, K, D, nat.F32, D))
    ref = torch.empty(n, dtype=torch.int64, device="cuda")
    nat.call("xgs_vq_assign", nat.ptr(x), nat.F32, n, D, D, nat.ptr(E), K, nat.ptr(ref), nat.ptr(ws), ws.numel(),
             None, nat.stream_ptr())
    for cnt in (0, 1, 1234, n, n + 500):
        codes = torch.full((n,), -7, dtype=torch.int64, device="cuda")
        n_dev = torch.tensor([cnt], dtype=torch.int64, device="cuda")
        nat.call("xgs_vq_assign_dev", nat.ptr(x), nat.F32, n, D, D, nat.ptr(E), K, nat.ptr(codes), nat.ptr(ws),
                 ws.numel(), nat.ptr(n_dev), nat.stream_ptr())
        m = min(cnt, n)
        assert torch.equal(codes[:m], ref[:m]), cnt
        assert bool((codes[m:] == -7).all()), cnt
