"""Pin the CPU oracle against the reference's golden vectors and its own KATs.

The fixtures in tests/golden were produced by the reference itself
(tests/golden/make_golden.py); the KATs restate pkg/tests/test_vq.py.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import grid as og
from oracle import native as on
from oracle import vq as ov


def test_sqdist_numpy_and_c_match_reference():
    g = golden("sqdist")
    for D in (1, 3, 7, 8, 9, 17, 100, 128, 129, 255, 512, 768, 1152):
        x, E, d = g[f"x_{D}"], g[f"E_{D}"], g[f"d_{D}"]
        assert np.array_equal(ov.squared_distances(x, E), d)
        assert np.array_equal(on.sqdist(x, E), d)


def test_pairwise_sum_model():
    rng = np.random.default_rng(0)
    for n in (0, 1, 5, 8, 9, 127, 128, 129, 300, 512, 1000, 1152):
        a = rng.normal(size=n) ** 2
        assert on.pairwise_sum(a) == np.sum(a)


def test_assign_matches_reference():
    g = golden("assign")
    for case in ("c1", "c2", "tie", "tie2"):
        x, E, codes = g[f"{case}_x"], g[f"{case}_E"].astype(np.float64), g[f"{case}_codes"]
        assert np.array_equal(ov.assign_batch(x, E), codes)
        assert np.array_equal(on.assign(x, E, threads=2), codes)
    assert list(g["tie_codes"][:3]) == [3, 3, 3]


def test_accumulate_ema_match_reference():
    g = golden("accumulate")
    x, E = g["x"], g["E"]
    counts, sums = ov.accumulate(x, E)
    assert np.array_equal(counts, g["counts"]) and np.array_equal(sums, g["sums"])
    c2, s2 = on.accumulate(x, on.assign(x, E), E.shape[0])
    assert np.array_equal(c2, g["counts"]) and np.array_equal(s2, g["sums"])
    cb = ov.OracleCodebook(E, g["N0"], g["M0"], 0.99, 1e-5)
    e = ov.ema_step(cb, g["counts"], g["sums"])
    assert np.array_equal(e.N, g["N1"]) and np.array_equal(e.M, g["M1"])
    assert np.array_equal(e.E, g["E1"])


def test_online_step_sequences_match_reference():
    g = golden("online")
    cb = ov.OracleCodebook(g["a_E0"], np.zeros(4), np.zeros((4, 3)), 0.8, 1e-5,
                           ov.OracleReservoir(128, 3))
    rng = np.random.default_rng(7)
    for i, b in enumerate(g["a_batches"]):
        cb, rev, _ = ov.online_step(cb, b, 0.7, 0.5, 1e-2, rng)
        assert np.array_equal(cb.E, g["a_E"][i]) and np.array_equal(cb.N, g["a_N"][i])
        assert len(rev) == g["a_nrev"][i]
    assert g["a_nrev"].sum() > 0  # the fixture exercises revival
    K = 64
    cb = ov.OracleCodebook(g["b_E0"], np.zeros(K), np.zeros((K, 32)), 0.99, 1e-5,
                           ov.OracleReservoir(300, 32))
    rng = np.random.default_rng(12)
    x = g["b_x"]
    for i in range(8):
        cb, rev, _ = ov.online_step(cb, x[i * 256:(i + 1) * 256], 0.7, 0.5 / K, 1e-3, rng,
                                    assume_all_pass=True)
        assert np.array_equal(cb.E, g["b_E"][i]) and np.array_equal(cb.N, g["b_N"][i])
        assert len(rev) == g["b_nrev"][i]


def test_confidence_and_warm_start_match_reference():
    g = golden("online")
    p = ov.confidence_scores(g["c_x"], g["c_E"], 0.7)
    assert np.array_equal(p, g["c_p"])
    assert np.array_equal(ov.confidence_mask(g["c_x"], g["c_E"], 0.7, 0.4), g["c_mask"])
    seeds = ov.seed_from_samples(g["d_buf"], 4)
    assert np.array_equal(seeds, g["d_seeds"])
    cb = ov.OracleCodebook(seeds, np.zeros(4), np.zeros((4, 3)), 0.96, 1e-5)
    out, used, degen = ov.warm_start(g["d_buf"], cb, 0.7, 0.3)
    assert not degen and used == int(g["d_used"])
    assert np.array_equal(out.E, g["d_E"]) and np.array_equal(out.N, g["d_N"])


# ---- restated reference KATs (pkg/tests/test_vq.py) ----

def test_kat_tie_breaks_low():  # test_vq.py:34-36
    assert ov.assign_batch(np.array([[1.0]]), np.array([[0.0], [2.0]]))[0] == 0


def test_kat_monotone_decay_exact():  # test_vq.py:103-114
    cb = ov.OracleCodebook(np.zeros((4, 2)), np.array([1.0, 2.0, 0.5, 7.0]), np.zeros((4, 2)),
                           0.96, 1e-5)
    ref = cb.N.copy()
    for _ in range(30):
        cb = ov.ema_step(cb, np.zeros(4), np.zeros((4, 2)))
        ref = 0.96 * ref
        assert np.array_equal(cb.N, ref)


def test_kat_revive_value():  # test_vq.py:223-232
    cb = ov.OracleCodebook(np.ones((2, 2)), np.array([1.0, 0.0]), np.zeros((2, 2)), 0.96, 1e-5,
                           ov.OracleReservoir(64, 2))
    v = np.array([3.0, -1.0])
    cb.reservoir.extend(v[None])
    out, rev, skipped = ov.revive_dead_codes(cb, 1e-2, np.random.default_rng(0))
    assert rev == [1] and not skipped
    assert np.allclose(out.E[1], v / (1 + 2e-5)) and out.N[1] == 1 + 1e-5


# ---- back-projection + grid ----

def test_backproject_matches_reference_bits():
    g = golden("backproject")
    R, t, pid = g["R"], g["t"], g["pose_id"]
    for k in range(R.shape[0]):
        sel = pid == k
        p = on.backproject(R[k], t[k], g["intr"], g["u"][sel], g["v"][sel],
                           g["d"][sel].astype(np.float64))
        assert np.array_equal(p, g["p"][sel])


def test_grid_key_kats():
    # identity pose, hand-computed keys: pixel (u,v)=(0,0), depth 1, f=1, c=0
    depth = np.zeros((4, 4), np.float32)
    depth[0, 0] = 1.0           # p = (0,0,1) -> voxel (0,0,10) at vs=0.1
    depth[2, 3] = 0.5           # p = (1.0, 1.5, 0.5) -> (10, 15, 5)
    depth[1, 1] = -1.0          # invalid
    intr = np.array([1.0, 1.0, 0.0, 0.0])
    keys, pts = on.grid_keys(depth, intr, np.eye(3), np.zeros(3), 0.1)
    assert keys[0] == og.pack_key(0, 0, 10) and keys[11] == og.pack_key(10, 15, 5)
    assert (keys == og.KEY_INVALID).sum() == 14
    # floor semantics on exact boundaries and negatives
    depth = np.zeros((1, 2), np.float32)
    depth[0, 1] = 0.25
    keys, _ = on.grid_keys(depth, np.array([1.0, 1.0, 0.0, 2.0]), np.eye(3), np.zeros(3), 0.25)
    # v=1, cy=2 -> y = (1-2)*0.25 = -0.25 -> floor(-1.0) = -1 ; z = 0.25 -> 1
    assert keys[1] == og.pack_key(0, -1, 1)
    assert og.unpack_key(og.pack_key(-5, 7, -1048576)) == (-5, 7, -1048576)


def test_grid_first_pick_and_occupancy():
    depth = np.full((2, 3), 1.0, np.float32)
    color = np.arange(18, dtype=np.uint8).reshape(2, 3, 3)
    intr = np.array([100.0, 100.0, 0.0, 0.0])
    occ = set()
    out = og.grid_sample([(depth, color, np.eye(3), np.zeros(3))], intr, 1.0, occ)
    # every pixel lands in voxel (0,0,1): the lowest pixel id wins
    assert out["pid"].tolist() == [0] and len(occ) == 1
    assert np.array_equal(out["color"][0], color[0, 0] / 255.0)
    again = og.grid_sample([(depth, color, np.eye(3), np.zeros(3))], intr, 1.0, occ)
    assert again["pid"].size == 0  # pre-occupied voxel -> rejected
    m = og.grid_sample([(depth, color, np.eye(3), np.zeros(3))], intr, 1.0, set(), mode="mean")
    assert m["count"][0] == 6
