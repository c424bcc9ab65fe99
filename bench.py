"""Benchmark of the X-GS hot path on B200 (driver contract: one JSON line).

Headline workload = BASELINE.json configs[1] ("VQ at scale"): per GPU, a
resident batch of N = 1,048,576 fp32 unit-norm D=512 features from a
1024-centre mixture (sigma 0.05), codebook K = 1024, lam 0.99, delta 1e-3,
gamma 0.5/K (mask provably all-true); one step = one
online_step (reservoir, assign, accumulate, EMA, revival) over the batch.
Weak scaling: each rank holds its own 1,048,576-row shard and the per-code
stats are combined with one NCCL all-reduce per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import os

# NumPy's OpenBLAS threads keep spinning after a BLAS call in the CPU legs and
# take the host cores from the thread that drives the GPU (a rasterizer build
# right after a CPU leg read 88-136 ms instead of 1.3 ms).  The NumPy parts of
# the CPU baselines are single-threaded (their "cores": 1); the C port runs
# its own threads.
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import gc
import json
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ROWS, D, K, CENTRES, SIGMA = 1 << 20, 512, 1024, 1024, 0.05
LAM, DELTA, EPS, CAP = 0.99, 1e-3, 1e-5, 4096
METRIC = "VQ Mfeat/s (online_step: assign + accumulate + EMA + revival)"
WORKLOAD = "C2: VQ at scale, N=1048576/GPU x D=512 fp32, K=1024, lam=0.99, delta=1e-3, gamma=0.5/K"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: an NVML
    polling thread (10 ms period: short timed regions still get samples, negligible GIL load);
    nvidia-smi -lms as the fallback when NVML is unavailable."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, index):
        self.index, self.sm, self.mx, self.reasons = index, [], None, set()
        self.stop_evt = threading.Event()
        self.thread = None
        self.nvml = None

    def _handle(self, nv):
        try:
            import torch
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = self._handle(nv)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            self.nvml = nv

            def poll():
                while not self.stop_evt.is_set():
                    try:
                        self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                        r = get_r(h)
                        for nm, bit in self.REASONS:
                            if r & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    time.sleep(0.01)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
        except Exception:
            self.nvml = None
            self._smi_start()

    def _smi_start(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        self.lines = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=lambda: self.lines.extend(ln.strip() for ln in self.proc.stdout),
                             daemon=True).start()
        except OSError:
            self.proc = None

    def stop(self):
        if self.nvml is not None:
            self.stop_evt.set()
            self.thread.join(1.0)
            return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.mx,
                    "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}
        if getattr(self, "proc", None) is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for (nm, _), v in zip(self.REASONS, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi"}


def make_data(torch, rank, device):
    """Seeded synthetic mixture on the device (centres / E0 shared by all ranks)."""
    g = torch.Generator(device=device)
    g.manual_seed(10)
    C = torch.randn(CENTRES, D, generator=g, device=device, dtype=torch.float32)
    C /= C.norm(dim=1, keepdim=True)

    def sample(n, seed):
        g.manual_seed(seed)
        out = torch.empty(n, D, device=device, dtype=torch.float32)
        for s in range(0, n, 1 << 18):
            m = min(1 << 18, n - s)
            ids = torch.randint(0, CENTRES, (m,), generator=g, device=device)
            v = C[ids] + SIGMA * torch.randn(m, D, generator=g, device=device)
            out[s:s + m] = v / v.norm(dim=1, keepdim=True)
        return out

    x = sample(N_ROWS, 100 + rank)
    E0 = sample(K, 11).double()
    return x, E0


FP64_DMMA_TFLOPS = 37.1   # tools/micro/fp64_peak.cu on the B200 pool (profiles/r2_fp64_peak_microbench.txt)
GRID_F, GRID_H, GRID_W = 16, 720, 1280
GRID_INTR = (1050.0, 1050.0, 359.5, 639.5)   # BASELINE leaves C3 intrinsics open
GRID_MAP = 4_000_000
# the scene map's hash set: 16M slots (128 MB) for the 4M voxels plus a batch's new ones at load
# <= 1/2 (the library reserves room for min(pixels, batch-table slots) new keys per batch)
GRID_MAP_SLOTS = 4 * GRID_MAP


def grid_scene_objects(seed=20):
    from paper_2603_09632_b200 import synth
    rng = np.random.default_rng(seed)
    planes = synth.random_planes(rng, 6, spread=3.0)
    spheres = [(rng.uniform(-1.0, 1.0, 3), rng.uniform(0.2, 0.6)) for _ in range(4)]
    return planes, spheres


def grid_scene(seed=20, frames=GRID_F):
    """C3: 16 frames 1280x720, random planes + spheres 0.3-8 m, sigma 3 mm,
    circle of radius 2 m with 5 deg yaw steps, uint8 colour (seeds 20/21)."""
    from paper_2603_09632_b200 import synth
    planes, spheres = grid_scene_objects(seed)
    poses = synth.circle_trajectory(frames, radius=2.0, step_deg=5.0)
    crng = np.random.default_rng(seed + 1)
    D = np.empty((frames, GRID_H, GRID_W), np.float32)
    C = np.empty((frames, GRID_H, GRID_W, 3), np.uint8)
    for i, p in enumerate(poses):
        D[i], C[i] = synth.rgbd_frame(crng, p, GRID_INTR, GRID_H, GRID_W, planes=planes, spheres=spheres,
                                      dmin=0.3, dmax=8.0, noise=0.003, zero_frac=0.0)
    R = np.stack([p.rotation for p in poses])
    T = np.stack([p.translation for p in poses])
    return D, C, R, T


def grid_warm_map(torch, voxel, target=GRID_MAP, seed=20, max_frames=240):
    """The C3 running map: voxels of the SAME scene seen earlier along the
    trajectory -- the rest of the 2 m circle (yaw 80..355 deg), then rings at
    other heights and radii -- sampled by GridSampler itself at `voxel`, until
    ~`target` voxels or `max_frames` frames (1 cm reaches ~4M; at 5 cm the
    scene holds far fewer voxels, so seeded filler keys far outside the scene
    volume bring the hash set to ~`target`).  Returns (uint64-as-int64 CUDA
    keys, scene voxel count, frames used)."""
    from paper_2603_09632_b200 import synth
    from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet, pack_key
    planes, spheres = grid_scene_objects(seed)
    rings = [(2.0, 0.0, 80.0), (2.0, 0.6, 0.0), (2.6, -0.5, 0.0), (1.4, 0.3, 0.0), (3.0, 1.0, 0.0), (2.3, -1.0, 0.0)]
    hs = VoxelHashSet(2 * target + (1 << 22))
    gs = GridSampler(GRID_INTR, voxel, occupied=hs)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed + 2)
    keys, used = [], 0
    for radius, height, a0 in rings:
        poses = []
        a = a0
        while a < 360.0 and used + len(poses) < max_frames:
            eye = np.array([radius * np.cos(np.deg2rad(a)), radius * np.sin(np.deg2rad(a)), height])
            poses.append(synth.look_at(eye, np.zeros(3)))
            a += 5.0
        for i in range(0, len(poses), 16):
            chunk = poses[i:i + 16]
            R = torch.tensor(np.stack([p.rotation for p in chunk]), device="cuda")
            T = torch.tensor(np.stack([p.translation for p in chunk]), device="cuda")
            D = torch.stack([synth.render_depth_torch(torch, R[j], T[j], GRID_INTR, GRID_H, GRID_W, planes, spheres)
                             for j in range(len(chunk))])
            D = torch.where(D > 0, D + 0.003 * torch.randn(D.shape, generator=g, device="cuda", dtype=D.dtype), D)
            r = gs.sample(D.float().contiguous(), (R, T))
            keys.append(r.key.clone())
            used += len(chunk)
            if sum(int(k.numel()) for k in keys) >= target:
                break
        if sum(int(k.numel()) for k in keys) >= target or used >= max_frames:
            break
    scene = torch.cat(keys)
    n_scene = int(scene.numel())
    hs.close()
    if n_scene < target:   # filler: seeded keys at |index| in [1e5, 2e5) voxels -- outside any batch's reach
        rng = np.random.default_rng(seed + 3)
        m = target - n_scene
        q = rng.integers(100_000, 200_000, (m, 3)) * rng.choice([-1, 1], (m, 3))
        scene = torch.cat([scene, torch.from_numpy(pack_key(q[:, 0], q[:, 1], q[:, 2]).view(np.int64)).cuda()])
    return scene, n_scene, used


def grid_graph_times(torch, voxel, warm, frames, steps, ref):
    """The same C3 batch through GridGraph (XGS_GRID_ASYNC captured in a CUDA
    graph): one graph launch, kernels back to back with no host work between
    them.  The map is restored from a snapshot (VoxelHashSet.copy_from, outside
    the timed region) before every replay, so each replay sees the ~4M-voxel
    running map; CUDA events around the replay on its stream."""
    from paper_2603_09632_b200.grid import GridGraph, GridSampler, VoxelHashSet
    Dd, Rd, Td, Cd = frames
    npix = int(Dd.numel())
    snap = VoxelHashSet(GRID_MAP_SLOTS)
    snap.insert(warm)
    work = VoxelHashSet(GRID_MAP_SLOTS)
    work.copy_from(snap)
    gg = GridGraph(GridSampler(GRID_INTR, voxel, occupied=work), Dd, (Rd, Td), Cd)
    times = []
    res = None
    for it in range(steps + 1):
        work.copy_from(snap)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gg.replay()
        e1.record()
        torch.cuda.synchronize()
        res = gg.result()
        if it > 0:
            times.append(e0.elapsed_time(e1))
    same = (len(res) == len(ref) and res.n_voxels == ref.n_voxels and
            bool(torch.equal(res.key, ref.key)) and bool(torch.equal(res.pid, ref.pid)))
    snap.close()
    work.close()
    return {"ms_per_batch": float(np.median(times)), "new_voxels": len(res), "matches_sync_call": same}


def run_grid(torch, steps, cpu=True):
    """C3 grid sampling: Mpts/s = 16*1280*720 input pixels / batch time, map
    reset to the scene-derived ~4M-voxel running map before every timed batch."""
    from paper_2603_09632_b200 import _native as nat
    from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet
    D, C, R, T = grid_scene()
    Dd, Cd = torch.from_numpy(D).cuda(), torch.from_numpy(C).cuda()
    Rd, Td = torch.from_numpy(R).cuda(), torch.from_numpy(T).cuda()
    out = {}
    npix = GRID_F * GRID_H * GRID_W
    pk_, _ = peaks()
    for voxel in (0.01, 0.05):
        warm, n_scene, warm_frames = grid_warm_map(torch, voxel)
        times, calls, spans, stage = [], [], [], {}
        r = None
        # iterations 1..steps: the batch span alone (profile_only: no events between its
        # kernels, so the launches chain as in production); then `steps` more with every
        # stage scope for the per-stage split
        for it in range(2 * steps + 1):
            staged = it > steps
            hs = VoxelHashSet(GRID_MAP_SLOTS)
            hs.insert(warm)
            map_size = len(hs)
            gs = GridSampler(GRID_INTR, voxel, occupied=hs)
            torch.cuda.synchronize()
            nat.profile_only(None if staged else "grid_batch")
            nat.profile_enable(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            r = gs.sample(Dd, (Rd, Td), Cd)
            e1.record()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            prof = {t: nat.profile_read(t)[0] for t in ("grid_batch", "grid_keys", "grid_select", "grid_emit")}
            nat.profile_enable(False)
            nat.profile_only(None)
            if it > 0 and not staged:   # the first batch sizes the library's tables
                times.append(e0.elapsed_time(e1))
                calls.append((t1 - t0) * 1e3)
                spans.append(prof["grid_batch"])
            if staged:
                for k_, v_ in prof.items():
                    stage.setdefault(k_, []).append(v_)
            hs.close()
        ms = float(np.median(spans))
        stage_ms = {k_: float(np.median(v_)) for k_, v_ in stage.items()}
        n_new, n_vox = len(r), r.n_voxels
        graph = grid_graph_times(torch, voxel, warm, (Dd, Rd, Td, Cd), steps, r)
        # algorithmic bytes of the batch: depth in (4 B/px) + colour of the new voxels' pixels (3 B) + the
        # outputs written (key 8, pid 8, mu 24, colour 24, scale 8, depth 8, count 8 = 88 B per new voxel)
        # + one 32 B map-table sector per distinct voxel of the batch
        batch_bytes = 4.0 * npix + n_new * (3 + 88) + 32.0 * n_vox
        front_bytes = 4.0 * npix          # the front end's compulsory HBM traffic (depth read)
        t_front = stage_ms["grid_keys"]
        # end to end through the public API: frames in pinned host memory (H2D of depth + colour),
        # the batch, the new Gaussians back to host numpy (GridSampleResult.to_numpy)
        Dh, Ch = torch.from_numpy(D).pin_memory(), torch.from_numpy(C).pin_memory()
        e2e = []
        for it in range(3):
            hs = VoxelHashSet(GRID_MAP_SLOTS)
            hs.insert(warm)
            gs = GridSampler(GRID_INTR, voxel, occupied=hs)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            host_out = gs.sample(Dh, (Rd, Td), Ch).to_numpy()
            e2e.append((time.perf_counter() - t0) * 1e3)
            hs.close()
        e2e_ms = float(np.median(e2e))
        e2e_h2d = Dh.numel() * 4 + Ch.numel()
        e2e_d2h = sum(v.nbytes for v in host_out.values() if isinstance(v, np.ndarray))
        out[str(voxel)] = {
            "Mpts_per_s": npix / (ms * 1e-3) / 1e6, "ms_per_batch": ms,
            "ms_per_batch_python_call": float(np.median(calls)), "ms_per_batch_events": float(np.median(times)),
            "pixels": npix, "valid_points": r.n_valid, "batch_voxels": n_vox, "new_voxels": n_new,
            "rejected_voxels": n_vox - n_new, "rejected_frac": (n_vox - n_new) / max(1, n_vox),
            "map_voxels_before": map_size, "map_scene_voxels": n_scene, "map_warm_frames": warm_frames,
            "items_inserted": r.n_sorted, "per_stage_ms": stage_ms, "graph": graph,
            "batch_hbm_frac": batch_bytes / (ms * 1e-3) / 1e9 / pk_["hbm_gbs"],
            "roofline": {"bound": "hbm", "kernel": "grid_front_kernel<FRONT_INSERT> (back-projection, keys, "
                                                   "left/up dedup, batch-table insert)",
                         "achieved": front_bytes / (t_front * 1e-3) / 1e9, "peak": pk_["hbm_gbs"], "unit": "GB/s",
                         "frac": front_bytes / (t_front * 1e-3) / 1e9 / pk_["hbm_gbs"],
                         "algorithmic_bytes": front_bytes,
                         "traffic": (ncu_traffic("grid_front_kernel_C3_1cm") if voxel == 0.01 else None),
                         "issue": grid_issue_roofline(),
                         "note": "issue/L2-latency bound: fp32 key filter + ballot staging per pixel, one random "
                                 "L2 sector per inserted item (tools/micro/insert_bench.cu: ~35 us floor for 4.4M "
                                 "probes even read-only)"},
            "e2e": {"Mpts_per_s": npix / (e2e_ms * 1e-3) / 1e6, "ms_per_batch": e2e_ms,
                    "h2d_bytes": e2e_h2d, "d2h_bytes": e2e_d2h,
                    "note": "host wall clock around sample() + to_numpy(), pinned host frames"}}
    out["timing"] = ("ms_per_batch = device span of the C-ABI call xgs_grid_sample (first launch .. its status "
                     "sync; ProfScope 'grid_batch' recorded alone, no events between the kernels); per_stage_ms "
                     "from separate batches with every stage scope on; ms_per_batch_python_call adds the Python "
                     "wrapper")
    if cpu:
        from oracle import grid as og
        t0 = time.perf_counter()
        nf = 2
        og.grid_sample([(D[i], C[i], R[i], T[i]) for i in range(nf)], np.array(GRID_INTR), 0.01, set())
        el = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": nf * GRID_H * GRID_W / el / 1e6, "unit": "Mpts/s", "cores": 1,
                               "kind": "port", "sample": f"{nf} C3 frames, voxel 0.01, oracle/grid.py "
                                                         "(C back-projection + NumPy sort/unique/isin)"}
    return out


STREAM_H, STREAM_W, STREAM_D, STREAM_K = 480, 640, 768, 512
STREAM_INTR = (525.0, 525.0, 239.5, 319.5)


def run_c1(torch, reps=20, cpu=True):
    """C1 (BASELINE configs[0], the reference's CPU-runnable case): one 640x480
    frame (6 planes 0.5-5 m, sigma 5 mm, 5% zeros, fx=fy=525, identity pose),
    grid sampling at 0.02 m into an empty map, one 512-dim unit-norm feature
    per new point (64-centre mixture, sigma 0.1), K=256 codebook from random
    rows of them, one online_step (lam 0.99).  Latency = host wall clock of
    GridSampler.sample + online_step on device-resident inputs (median of
    `reps`; fresh map each time), and the same through the CPU port."""
    from paper_2603_09632_b200 import synth
    from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet
    import paper_2603_09632_b200 as xv
    d, col, pose, intr4 = synth.config1_frame(0)
    dd, cd = torch.from_numpy(d).cuda(), torch.from_numpy(col).cuda()
    R = torch.from_numpy(pose.rotation[None].copy()).cuda()
    T = torch.from_numpy(pose.translation[None].copy()).cuda()
    probe = GridSampler(intr4, 0.02).sample(dd, (R, T), cd)
    n = len(probe)
    rng = np.random.default_rng(2)
    x = synth.mixture_features(rng, n, 512, 64, 0.1)
    E0 = x[np.random.default_rng(3).choice(n, 256, replace=False)].astype(np.float64)
    xd = torch.from_numpy(x).cuda()
    cfg = xv.VqConfig(K=256, lam=0.99, gamma=0.5 / 256, delta_dead=1e-3)
    times = []
    for _ in range(reps + 3):
        hs = VoxelHashSet(1 << 20)
        gs = GridSampler(intr4, 0.02, occupied=hs)
        cb = xv.Codebook._make(torch.from_numpy(E0).cuda(), torch.zeros(256, dtype=torch.float64, device="cuda"),
                               torch.zeros(256, 512, dtype=torch.float64, device="cuda"), 0.99, 1e-5,
                               xv.FeatureReservoir(4096, 512))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = gs.sample(dd, (R, T), cd)
        cb, _ = xv.online_step(cb, xd[:len(r)], cfg, np.random.default_rng(4))
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
        hs.close()
    ms = float(np.median(times[3:]))
    out = {"ms_per_frame_step": ms, "new_gaussians": n, "pixels": d.size,
           "workload": "C1: one 640x480 RGB-D frame (6 planes 0.5-5 m), grid 0.02 m, K=256 D=512 online_step on the "
                       "new points' features; host wall clock of GridSampler.sample + online_step"}
    if cpu:
        from oracle import grid as og
        from oracle import native as on
        from oracle import vq as ov
        t0 = time.perf_counter()
        og.grid_sample([(d, col, pose.rotation, pose.translation)], np.array(intr4), 0.02, set())
        oc = ov.OracleCodebook(E0, np.zeros(256), np.zeros((256, 512)), 0.99, 1e-5, ov.OracleReservoir(4096, 512))
        oc.reservoir.extend(x)
        codes = on.assign(x, oc.E, threads=1)
        counts, sums = on.accumulate(x, codes, 256)
        oc = ov.ema_step(oc, counts, sums)
        ov.revive_dead_codes(oc, 1e-3, np.random.default_rng(4))
        el = (time.perf_counter() - t0) * 1e3
        out["cpu_baseline"] = {"ms_per_frame_step": el, "cores": 1, "kind": "port",
                               "sample": "the whole C1 step: oracle/grid.py (C back-projection + NumPy voxel "
                                         "dedup) + online_step with the C assign/accumulate (1 thread)"}
    return out


STREAM_FEAT_HW = (60, 80)     # VFM-resolution feature map (stride 8 on 480x640)


def run_stream(torch, frames, device):
    """C4: 1000 frames of 640x480 RGB-D -- 8 static walls 3-7 m away plus two
    fresh random spheres 1.2-2.6 m away per frame (new surface entering the view: ~2K new
    voxels per frame, so the map grows to ~2M), random-walk poses (1 cm / 1
    deg step sigma), depth noise 5 mm, 5% invalid pixels -- each grid-sampled
    at 0.02 m into new Gaussians whose 768-dim features are gathered from the
    frame's (768, 60, 80) feature map (512-centre mixture) and fed to online
    VQ with K=512, lam=0.99.  One frame = PerceiverStream.step (staging
    copies + one CUDA-graph replay + one small read-back + the host revival);
    per-frame latency is the host wall clock around it, p50 / p99."""
    from paper_2603_09632_b200 import synth
    from paper_2603_09632_b200.stream import PerceiverStream
    import paper_2603_09632_b200 as xv
    rng = np.random.default_rng(30)
    planes = synth.facing_planes(rng, 8, 3.0, 7.0)
    poses = synth.random_walk_trajectory(frames, rng, step_t=0.01, step_deg=1.0)
    g = torch.Generator(device=device)
    g.manual_seed(31)
    Cn = torch.randn(512, STREAM_D, generator=g, device=device)
    Cn /= Cn.norm(dim=1, keepdim=True)
    E0 = Cn[torch.randint(0, 512, (STREAM_K,), generator=g, device=device)] + 0.05 * torch.randn(
        STREAM_K, STREAM_D, generator=g, device=device)
    E0 = (E0 / E0.norm(dim=1, keepdim=True)).double()
    cfg = xv.VqConfig(K=STREAM_K, lam=0.99, gamma=0.5 / STREAM_K, delta_dead=1e-3)
    cb = xv.Codebook._make(E0, torch.zeros(STREAM_K, dtype=torch.float64, device=device),
                           torch.zeros(STREAM_K, STREAM_D, dtype=torch.float64, device=device), 0.99, 1e-5,
                           xv.FeatureReservoir(cfg.reservoir_capacity, STREAM_D))
    Hf, Wf = STREAM_FEAT_HW
    st = PerceiverStream(STREAM_INTR, STREAM_H, STREAM_W, 0.02, cb, cfg, (STREAM_D, Hf, Wf),
                         np.random.default_rng(32), map_capacity=1 << 23, vq_capacity=8192)
    noise = torch.Generator(device=device)
    noise.manual_seed(33)
    lat, newpts, graph = [], [], 0
    for i, p in enumerate(poses):
        R = torch.tensor(p.rotation, device=device)
        t = torch.tensor(p.translation, device=device)
        c = p.camera_center()
        sph = [(c + p.rotation.T @ np.array([rng.uniform(-0.8, 0.8), rng.uniform(-1.0, 1.0), rng.uniform(1.2, 2.6)]),
                rng.uniform(0.22, 0.4)) for _ in range(2)]
        d = synth.render_depth_torch(torch, R, t, STREAM_INTR, STREAM_H, STREAM_W, planes, sph)
        d = d + 0.005 * torch.randn(d.shape, generator=noise, device=device, dtype=torch.float64) * (d > 0)
        d = torch.where(torch.rand(d.shape, generator=noise, device=device) < 0.05, torch.zeros_like(d), d)
        d = d.float().contiguous()
        col = torch.randint(0, 256, (STREAM_H, STREAM_W, 3), generator=noise, device=device, dtype=torch.uint8)
        f = Cn[torch.randint(0, 512, (Hf * Wf,), generator=noise, device=device)] + 0.05 * torch.randn(
            Hf * Wf, STREAM_D, generator=noise, device=device)
        f = (f / f.norm(dim=1, keepdim=True)).T.reshape(STREAM_D, Hf, Wf).contiguous()
        # the frame arrives in the stream's staging buffers (the sensor / feature
        # producer writes them), then one step
        sd, sR, sT, sc, sf = st.inputs()
        sd.view(-1).copy_(d.reshape(-1))
        sR.view(-1).copy_(R.reshape(-1))
        sT.view(-1).copy_(t.reshape(-1))
        sc.view(-1).copy_(col.reshape(-1))
        sf.view(-1).copy_(f.reshape(-1))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = st.step(sd, (sR, sT), sc, sf)
        lat.append((time.perf_counter() - t0) * 1e3)
        newpts.append(r.n_new)
        graph += int(r.graph)
    lat = np.array(lat[5:])   # frame 1 sizes the library state and captures the graph
    return {"frames": frames, "p50_ms": float(np.percentile(lat, 50)), "p99_ms": float(np.percentile(lat, 99)),
            "mean_ms": float(lat.mean()), "frames_per_s": float(1e3 / lat.mean()),
            "map_voxels": int(sum(newpts)), "mean_new_per_frame": float(np.mean(newpts)),
            "max_new_per_frame": int(np.max(newpts)), "graph_frames": graph,
            "timing": "host wall clock around PerceiverStream.step with the frame already in the stream's staging "
                      "buffers: one CUDA-graph replay of grid sampling + VQ assign/accumulate/EMA, one read-back of "
                      "N + counts, reservoir write, revival",
            "workload": "C4: 640x480 RGB-D (8 static walls 3-7 m + 2 fresh random spheres per frame), random-walk "
                        "poses (1 cm / 1 deg), grid 0.02 m, 768-dim features gathered from a 60x80 map per frame "
                        "(512-centre mixture), VQ K=512 lam=0.99 on the new points"}


C5_TOTAL, C5_D, C5_K, C5_CENTRES = 67_108_864, 1152, 4096, 4096
C5_WORKLOAD = ("C5: multi-GPU VQ, N=67,108,864 rows in total x D=1152 bf16 (fp64-exact assignment), K=4096, "
               "lam=0.99, delta=1e-3, gamma=0.5/K; rows sharded across the ranks (strong scaling)")


def c5_data(torch, rank, world, device):
    """This rank's contiguous shard of the C5 batch, generated on the device
    (4096-centre unit-norm mixture, sigma 0.05, stored bf16; centres and the
    initial codebook are identical on every rank), plus E0 (K random rows of
    the same mixture, fp64)."""
    from paper_2603_09632_b200.distributed import strong_shard
    _, rows = strong_shard(C5_TOTAL, world, rank)
    g = torch.Generator(device=device)
    g.manual_seed(40)
    C = torch.randn(C5_CENTRES, C5_D, generator=g, device=device)
    C /= C.norm(dim=1, keepdim=True)
    x = torch.empty(rows, C5_D, device=device, dtype=torch.bfloat16)
    chunk = 1 << 20
    for s0 in range(0, rows, chunk):
        g.manual_seed(1_000_003 * (rank + 1) + s0 // chunk)    # per-(rank, chunk) stream
        m = min(chunk, rows - s0)
        v = C[torch.randint(0, C5_CENTRES, (m,), generator=g, device=device)] + 0.05 * torch.randn(
            m, C5_D, generator=g, device=device)
        x[s0:s0 + m] = (v / v.norm(dim=1, keepdim=True)).to(torch.bfloat16)
        del v
    g.manual_seed(41)
    e = C[torch.randint(0, C5_CENTRES, (C5_K,), generator=g, device=device)] + 0.05 * torch.randn(
        C5_K, C5_D, generator=g, device=device)
    E0 = (e / e.norm(dim=1, keepdim=True)).to(torch.bfloat16).double()
    del C, e
    torch.cuda.empty_cache()
    return x, E0


def run_c5(torch, iters, device):
    """C5 on ONE GPU (all 67,108,864 rows), for tools and the N=1 evidence:
    ms per online_step iteration and the per-stage split."""
    from paper_2603_09632_b200 import _native as nat
    from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
    import paper_2603_09632_b200 as xv
    x, E0 = c5_data(torch, 0, 1, device)
    cfg = xv.VqConfig(K=C5_K, lam=0.99, gamma=0.5 / C5_K, delta_dead=1e-3)
    vq = DataParallelVQ((E0, torch.zeros(C5_K, dtype=torch.float64, device=device),
                         torch.zeros(C5_K, C5_D, dtype=torch.float64, device=device)), cfg,
                        np.random.default_rng(41), CudaBackend(C5_K, C5_D, 0.99, 1e-5))
    vq.step(x, [x.shape[0]])
    torch.cuda.synchronize()
    nat.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        vq.step(x, [x.shape[0]])
    e1.record()
    torch.cuda.synchronize()
    prof = {t: nat.profile_read(t)[0] / iters for t in ("vq_prep", "vq_screen", "vq_rerank", "vq_accumulate",
                                                          "vq_chain", "vq_ema")}
    nat.profile_enable(False)
    ms = e0.elapsed_time(e1) / iters
    return {"rows": int(x.shape[0]), "iters": iters, "ms_per_iter": ms, "per_stage_ms": prof,
            "max_memory_allocated_GB": torch.cuda.max_memory_allocated() / 1e9,
            "device_memory_GB": torch.cuda.get_device_properties(device).total_memory / 1e9}


def run_targets(torch, iters, cpu=True):
    """grid-sampled supervision-target prefetch for one keyframe
    (480x640, stride 4 -> all 16 offsets, D=512 fp32 feature map at 1/16
    resolution), padded fp64 targets as the reference's SupervisionTarget."""
    from paper_2603_09632_b200 import _native as nat
    from paper_2603_09632_b200 import supervision as sup
    H, W, s, D = 480, 640, 4, 512
    g = torch.Generator(device="cuda")
    g.manual_seed(50)
    P = torch.randn(D, H // 16, W // 16, generator=g, device="cuda")
    src = sup.ContinuousFeatureSource(P)
    for _ in range(3):   # warm-up as the timed loop runs (two output sets alive at once: both blocks cached)
        G, V = sup.prefetch_targets(src, H, W, s, range(16))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        G, V = sup.prefetch_targets(src, H, W, s, range(16))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    nbytes = G.numel() * 8 + V.numel() * 8          # outputs dominate (the source is L2-resident)
    pk, _ = peaks()
    out = {"ms_per_keyframe": ms, "offsets": 16, "target_shape": list(G.shape), "GB_per_s": nbytes / (ms * 1e-3) / 1e9,
           "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
           "workload": "480x640 keyframe, stride 4 (16 offsets), D=512 continuous source at 30x40, fp64 targets"}
    del G, V
    if cpu:
        from oracle import supervision as osup
        Ph = P.double().cpu().numpy()
        t0 = time.perf_counter()
        for k in range(16):
            oh, ow = sup.next_offset(k, s, 0)
            Gc, Vc = osup.target_continuous(Ph, H, W, s, oh, ow)
            osup.pad(Gc, Vc, H, W, s)
        out["cpu_baseline"] = {"ms_per_keyframe": (time.perf_counter() - t0) * 1e3, "cores": 1, "kind": "port",
                               "sample": "the same 16 offsets through oracle/supervision.py (NumPy)"}
    return out


def run_init(torch, cpu=True):
    """codebook initialisation -- seed_from_samples (K-1
    farthest-point passes, queued without host syncs) then warm_start, on a
    16,384 x 512 fp32 buffer with the C2 codebook size K=1024."""
    import paper_2603_09632_b200 as xv
    n, D, K = 16384, 512, 1024
    g = torch.Generator(device="cuda")
    g.manual_seed(70)
    C = torch.randn(256, D, generator=g, device="cuda")
    lab = torch.randint(0, 256, (n,), generator=g, device="cuda")
    buf = C[lab] / C[lab].norm(dim=1, keepdim=True) + 0.05 * torch.randn(n, D, generator=g, device="cuda")
    buf = (buf / buf.norm(dim=1, keepdim=True)).contiguous()
    cfg = xv.VqConfig(K=K, gamma=0.5 / K)
    xv.seed_from_samples(buf[:1024], 8)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    seeds = xv.seed_from_samples(buf, K)
    e1.record()
    cb = xv.Codebook._make(seeds, torch.zeros(K, dtype=torch.float64, device="cuda"), torch.zeros_like(seeds), 0.99,
                           1e-5, xv.FeatureReservoir(16, D))
    ws = xv.warm_start(buf, cb, cfg)
    e2.record()
    torch.cuda.synchronize()
    ms_seed, ms_warm = e0.elapsed_time(e1), e1.elapsed_time(e2)
    step_bytes = n * D * 4 + n * 8 * 2                 # rows + min_d read/write per seed pass
    out = {"buffer_rows": n, "D": D, "K": K, "seed_ms": ms_seed, "seed_us_per_pass": ms_seed * 1e3 / (K - 1),
           "seed_pass_GB_per_s": step_bytes * (K - 1) / (ms_seed * 1e-3) / 1e9,
           "warm_start_ms": ms_warm, "warm_start_used": ws.used,
           "workload": "16384 x 512 fp32 unit-norm 256-centre mixture (seed 70), K=1024; the buffer is L2-resident"}
    if cpu:
        from oracle import vq as ov
        sample_k = 24
        bh = buf.cpu().numpy()
        t0 = time.perf_counter()
        ov.seed_from_samples(bh, sample_k)
        el = time.perf_counter() - t0
        out["cpu_baseline"] = {"seed_ms_extrapolated": el * 1e3 * (K - 1) / (sample_k - 1), "cores": 1,
                               "kind": "port", "sample": f"{sample_k} seeds through oracle/vq.py (NumPy), "
                                                         f"x{(K - 1) / (sample_k - 1):.1f} (cost is linear in K)"}
    del buf, seeds, cb, ws
    torch.cuda.empty_cache()
    return out


def run_consumers(torch, iters, cpu=True):
    """codebook consumers over a C4-sized map (about 2M
    Gaussians, K=512 logits, D=768 codebook): semantic_entropy (HBM-bound fused
    softmax + p log p over the fp64 logits), sample_tokens (entropy + stable
    descending radix sort + decode of the top M) and relevance_per_gaussian
    (decode = softmax rows + fp64 GEMM, then the contrast-score kernel)."""
    from paper_2603_09632_b200 import thinker as xt
    from paper_2603_09632_b200.core import Codebook, FeatureReservoir
    n, K, D, M = 1 << 21, 512, 768, 4096
    g = torch.Generator(device="cuda")
    g.manual_seed(60)
    L = torch.randn(n, K, generator=g, device="cuda", dtype=torch.float64) * 2.0
    E = torch.randn(K, D, generator=g, device="cuda", dtype=torch.float64)
    E = E / E.norm(dim=1, keepdim=True)
    cb = Codebook._make(E, torch.zeros(K, dtype=torch.float64, device="cuda"), E.clone(), 0.99, 1e-5,
                        FeatureReservoir(16, D))
    field = type("DeviceField", (), {"logits": L, "__len__": lambda self: n})()
    enc = xt.StubTextEncoder(D)
    q = xt.TextQuery.from_prompt("a chair", enc)

    def timed(fn, reps):
        fn()
        fn()   # two warm-up calls: the first touches freshly allocated scratch / output pages
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    pk, _ = peaks()
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    ms_h = timed(lambda: xt.semantic_entropy(L), iters)
    ent_bytes = n * K * 8 + n * 8
    ms_tok = timed(lambda: xt.sample_tokens(field, cb, M), max(1, iters // 2))
    ms_rel = timed(lambda: xt.relevance_per_gaussian(field, cb, q), 1)
    clocks = clk.stop()
    out = {"gaussians": n, "K": K, "D": D,
           "semantic_entropy": {"ms": ms_h, "GB_per_s": ent_bytes / (ms_h * 1e-3) / 1e9,
                                "hbm_frac": ent_bytes / (ms_h * 1e-3) / 1e9 / pk["hbm_gbs"],
                                "algorithmic_bytes": ent_bytes},
           "sample_tokens": {"ms": ms_tok, "M": M},
           "relevance_per_gaussian": {
               "ms": ms_rel, "fp64_TFLOPs": 2.0 * n * K * D / (ms_rel * 1e-3) / 1e12,
               "fp64_frac": 2.0 * n * K * D / (ms_rel * 1e-3) / 1e12 / FP64_DMMA_TFLOPS,
               "note": "softmax weights (xgs_softmax_rows) + xgs_gemm_f64 (DMMA.8x8x4 fp64, contrast fused in the "
                       "epilogue, no (n, D) features); frac vs the measured DMMA peak "
                       f"{FP64_DMMA_TFLOPS} TF/s (profiles/r2_fp64_peak_microbench.txt)"},
           "clocks": clocks,
           "workload": "2^21 Gaussians x K=512 fp64 logits (C4 map size), D=768 codebook, M=4096 tokens; "
                       "synthetic N(0, 2^2) logits"}
    if cpu:
        from oracle import thinker as ot
        Lh = L[:65536].cpu().numpy()
        t0 = time.perf_counter()
        ot.semantic_entropy(Lh)
        el = time.perf_counter() - t0
        out["cpu_baseline"] = {"semantic_entropy_ms_extrapolated": el * 1e3 * n / Lh.shape[0], "cores": 1,
                               "kind": "port", "sample": "65536 rows through oracle/thinker.py (NumPy), x32"}
    del L, E, cb, field
    torch.cuda.empty_cache()
    return out


def run_raster(torch, iters, cpu=True):
    """lattice rasterizer at keyframe scale -- 2^18 Gaussians
    in the frustum of a 480x640 camera, stride-4 lattice (120x160 pixels, the
    paper's grid-sampled semantic render), D=512 payload; build_blend_pairs,
    channel accumulation and the feature VJP timed separately."""
    from paper_2603_09632_b200 import rasterizer as rz
    from paper_2603_09632_b200.core import CameraIntrinsics, CameraPose
    from paper_2603_09632_b200.supervision import GridSpec
    n, H, W, s, D = 1 << 18, 480, 640, 4, 512
    g = torch.Generator(device="cuda")
    g.manual_seed(70)
    z = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 7.0 + 0.5
    u = (torch.rand(n, generator=g, device="cuda", dtype=torch.float64) - 0.5) * z * (H / 525.0)
    v = (torch.rand(n, generator=g, device="cuda", dtype=torch.float64) - 0.5) * z * (W / 525.0)
    q = torch.randn(n, 4, generator=g, device="cuda", dtype=torch.float64)
    field = type("DeviceField", (), {
        "mu": torch.stack([u, v, z], 1).contiguous(), "quat": (q / q.norm(dim=1, keepdim=True)).contiguous(),
        "scale": torch.exp(torch.rand(n, 3, generator=g, device="cuda", dtype=torch.float64) * 2.3 - 4.6),
        "opacity": torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 0.9 + 0.05,
        "color": torch.rand(n, 3, generator=g, device="cuda", dtype=torch.float64),
        "__len__": lambda self: n})()
    intr = CameraIntrinsics(fx=525.0, fy=525.0, cx=239.5, cy=319.5, height=H, width=W)
    pose = CameraPose.identity()
    grid = GridSpec(H=H, W=W, s=s)
    payload = torch.randn(n, D, generator=g, device="cuda", dtype=torch.float64)
    up = torch.randn(D, grid.H_s, grid.W_s, generator=g, device="cuda", dtype=torch.float64)

    def timed(fn, reps):
        """Median over `reps` calls, each bracketed by events (the build syncs on
        the host inside: one descheduled host thread must not skew a mean)."""
        fn()
        fn()   # two warm-up calls: the first touches freshly allocated scratch / output pages
        torch.cuda.synchronize()
        ts, r = [], None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts)), r

    ms_build, pr = timed(lambda: rz._Pairs(field, pose, intr, grid.rows(), grid.cols(), rz.DEFAULT_RASTER), iters)
    ms_acc, _ = timed(lambda: pr.accumulate(payload), iters)
    ms_vjp, _ = timed(lambda: pr.vjp(up.reshape(D, -1).contiguous(), D), iters)
    npairs, steps = pr.n_pairs, pr.blend_steps
    pr.close()
    pk, _ = peaks()
    # accumulate: pair metadata (4 + 8 B) + one D-row payload gather per alive pair (mostly L2 hits:
    # a splat's row is reused by every pixel it covers) + the (D, P) output; unique HBM bytes are the
    # metadata, the payload rows of the visible splats and the output
    acc_bytes = npairs * (4 + 8) + steps * D * 8 + grid.H_s * grid.W_s * D * 8
    hbm_bytes = npairs * (4 + 8) + grid.H_s * grid.W_s * D * 8
    out = {"gaussians": n, "lattice": [grid.H_s, grid.W_s], "D": D, "pairs": npairs, "blend_steps": steps,
           "build_ms": ms_build, "accumulate_ms": ms_acc, "vjp_ms": ms_vjp,
           "pairs_per_s": npairs / (ms_build * 1e-3),
           "accumulate_effective_GB_per_s": acc_bytes / (ms_acc * 1e-3) / 1e9,
           "accumulate_min_hbm_GB_per_s": hbm_bytes / (ms_acc * 1e-3) / 1e9,
           "accumulate_min_hbm_frac": hbm_bytes / (ms_acc * 1e-3) / 1e9 / pk["hbm_gbs"],
           "workload": "2^18 random Gaussians (0.5-8 m, 1-10 cm scales) in a 480x640 frustum, stride-4 lattice, "
                       "fp64 D=512 payload / cotangent"}
    del field, payload, up
    torch.cuda.empty_cache()
    return out


def cpu_port_rate(x_host, E, seconds=10.0, threads=None):
    """The reference's assign+accumulate restated in C (oracle/oracle.c), timed
    on host cores over row chunks until ~`seconds` elapse (bounded sample)."""
    from oracle import native as on
    threads = threads or os.cpu_count() or 1
    chunk = 64 * threads
    rows, t0 = 0, time.perf_counter()
    while True:
        lo = rows % (x_host.shape[0] - chunk)
        b = x_host[lo:lo + chunk]
        codes = on.assign(b, E, threads=threads)
        on.accumulate(b, codes, E.shape[0])
        rows += chunk
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return rows / el / 1e6, threads, rows, el


def c5_host_sample(n, seed=40):
    """A seeded host sample of the C5 distribution (4096-centre unit-norm
    mixture, sigma 0.05, bf16-rounded rows as uint16 bit patterns) and an
    initial codebook of K rows of it (fp64)."""
    import torch
    rng = np.random.default_rng(seed)
    C = rng.normal(size=(C5_CENTRES, C5_D))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    x = C[rng.integers(0, C5_CENTRES, n)] + 0.05 * rng.normal(size=(n, C5_D))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    xb = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)
    e = C[rng.integers(0, C5_CENTRES, C5_K)] + 0.05 * rng.normal(size=(C5_K, C5_D))
    e /= np.linalg.norm(e, axis=1, keepdims=True)
    E0 = torch.from_numpy(e.astype(np.float32)).to(torch.bfloat16).double().numpy()
    return xb.view(torch.int16).numpy().view(np.uint16), E0


def port_online_step(cb, xb, threads, rng):
    """The reference's online_step (vq.py:193-212) with the mask provably
    all-true (gamma = 0.5/K): assign + accumulate in the C restatement
    (oracle/oracle.c, fp64, NumPy pairwise order, `threads` host threads),
    reservoir extend, EMA and dead-code revival in NumPy (oracle/vq.py)."""
    from oracle import native as on
    from oracle import vq as ov
    import torch
    codes = on.assign(xb, cb.E, threads=threads, bf16=True)
    counts, sums = on.accumulate(xb, codes, cb.K, bf16=True)
    cb.reservoir.extend(torch.from_numpy(xb.view(np.int16)).view(torch.bfloat16).double().numpy())
    cb = ov.ema_step(cb, counts, sums)
    cb, _, _ = ov.revive_dead_codes(cb, DELTA, rng)
    return cb


def cpu_port_c5(seconds=10.0, threads=None):
    """C5 config on the host cores: port_online_step over chunks of 64 rows
    per thread until ~`seconds` elapse (bounded sample of the workload)."""
    from oracle import vq as ov
    threads = threads or os.cpu_count() or 1
    chunk = 64 * threads
    xs, E0 = c5_host_sample(max(4 * chunk, 8192))
    cb = ov.OracleCodebook(E0, np.zeros(C5_K), np.zeros((C5_K, C5_D)), LAM, EPS, ov.OracleReservoir(CAP, C5_D))
    rng = np.random.default_rng(42)
    cb = port_online_step(cb, xs[:chunk], threads, rng)      # warm (page-in, thread pool)
    rows, t0 = 0, time.perf_counter()
    while True:
        lo = (rows // chunk) % (xs.shape[0] // chunk) * chunk
        cb = port_online_step(cb, xs[lo:lo + chunk], threads, rng)
        rows += chunk
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": rows / el / 1e6, "unit": "Mfeat/s", "cores": threads, "kind": "port",
            "sample": f"{rows} rows of the C5 distribution in {el:.1f}s, {chunk} rows per online_step "
                      f"(assign+accumulate in oracle/oracle.c on {threads} threads, reservoir/EMA/revival in NumPy)"}


def reference_numpy_leg(seconds=20.0):
    """The UNMODIFIED reference's own semsplat.vq.online_step (baseline/_ref,
    NumPy, single-threaded) on C5-shaped batches of 8 rows (its (n, K, D) fp64
    broadcast temporary is 302 MB at 8 rows), timed for ~`seconds`."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "semsplat")):
        return None
    sys.path.insert(0, ref)
    try:
        from semsplat.core import Codebook, FeatureReservoir
        from semsplat.vq import VqConfig, online_step
    finally:
        sys.path.remove(ref)
    import torch
    xs, E0 = c5_host_sample(256)
    x = torch.from_numpy(xs.view(np.int16)).view(torch.bfloat16).double().numpy()
    cb = Codebook(E=E0, N=np.zeros(C5_K), M=np.zeros((C5_K, C5_D)), lam=LAM, epsilon=EPS,
                  reservoir=FeatureReservoir(CAP, C5_D))
    cfg = VqConfig(K=C5_K, lam=LAM, gamma=0.5 / C5_K, delta_dead=DELTA, epsilon=EPS, reservoir_capacity=CAP)
    rng = np.random.default_rng(42)
    b = 8
    cb, _ = online_step(cb, x[:b], cfg, rng)
    rows, t0 = 0, time.perf_counter()
    while True:
        lo = rows % (x.shape[0] - b)
        cb, _ = online_step(cb, x[lo:lo + b], cfg, rng)
        rows += b
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": rows / el / 1e6, "unit": "Mfeat/s", "cores": 1, "kind": "reference",
            "sample": f"{rows} rows of the C5 distribution through semsplat.vq.online_step (baseline/_ref, "
                      f"unmodified NumPy) in {b}-row batches, {el:.1f}s"}


def run_reference(args, rank, world):
    """--impl reference: the reference path's CPU implementation on the box's
    host cores for the headline config (C5): the C restatement of online_step
    (all host threads, 64 rows per thread per step), plus a labelled leg with
    the reference's own NumPy online_step."""
    if rank != 0:
        return
    from oracle import vq as ov
    threads = os.cpu_count() or 1
    chunk = 64 * threads
    xs, E0 = c5_host_sample(max(4 * chunk, 8192))
    cb = ov.OracleCodebook(E0, np.zeros(C5_K), np.zeros((C5_K, C5_D)), LAM, EPS, ov.OracleReservoir(CAP, C5_D))
    rng = np.random.default_rng(42)
    t_all, rows_all = 0.0, 0
    for it in range(args.warmup + args.steps):
        lo = (it * chunk) % (xs.shape[0] - chunk + 1)
        t0 = time.perf_counter()
        cb = port_online_step(cb, xs[lo:lo + chunk], threads, rng)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            t_all += dt
            rows_all += chunk
    v = rows_all / t_all / 1e6
    line = {"metric": "VQ Mfeat/s (online_step: assign + accumulate + EMA + revival), C5 strong scaling",
            "value": v, "unit": "Mfeat/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded 4096-centre unit-norm mixture, bf16-rounded)",
            "config": {"workload": C5_WORKLOAD, "cpu_rows_per_step": chunk},
            "cpu_baseline": {"value": v, "unit": "Mfeat/s", "cores": threads, "kind": "port",
                             "sample": f"{chunk} rows/step of the C5 distribution, K={C5_K}, D={C5_D}: "
                                       "oracle/oracle.c assign+accumulate + NumPy reservoir/EMA/revival "
                                       "(vq.py:193-212)"},
            "e2e": {"value": v, "unit": "Mfeat/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_cpu:
        line["reference_numpy"] = reference_numpy_leg(min(20.0, args.cpu_seconds * 2))
    print(json.dumps(line), flush=True)


def timed_steps(torch, vq, x, sizes, steps, barrier, world, device):
    """K timed online_steps bracketed by barrier + synchronize, CUDA events on
    the launching stream, max over ranks."""
    torch.cuda.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        vq.step(x, sizes)
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def profiled_steps(torch, vq, x, sizes, steps):
    from paper_2603_09632_b200 import _native as nat
    nat.profile_enable(True)
    for _ in range(steps):
        vq.step(x, sizes)
    torch.cuda.synchronize()
    prof = {t: nat.profile_read(t) for t in ("vq_prep", "vq_screen", "vq_rerank", "vq_accumulate", "vq_chain",
                                               "vq_ema")}
    nat.profile_enable(False)
    return prof


def grid_issue_roofline():
    """The grid front end is issue-bound, not HBM-bound: its instruction rate
    against the SM issue peak (4 warp instructions per SM per cycle at the max
    SM clock), from the committed ncu capture (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            v = json.load(f).get("grid_front_kernel_C3_1cm")
    except (OSError, ValueError):
        return None
    if not isinstance(v, dict):
        return None
    ach = v["warp_instructions"] / (v["duration_us"] * 1e-6)
    return {"achieved": ach, "peak": v["sm_issue_peak_warp_inst_per_s"], "unit": "warp inst/s",
            "frac": ach / v["sm_issue_peak_warp_inst_per_s"], "issue_active_pct": v["issue_active_pct"],
            "source": v["source"]}


def ncu_traffic(key):
    try:   # DRAM bytes of the screen kernel from a committed ncu capture (profiles/ncu_traffic.json)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            v = json.load(f).get(key)
        return v.get("bytes") if isinstance(v, dict) else v
    except (OSError, ValueError):
        return None


def screen_roofline(prof, flops_per_step, steps, traffic=None):
    pk, pk_kind = peaks()
    scr_ms, scr_n = prof["vq_screen"]
    # per step: the screen stage's event-timed span (main pass + rescreen of
    # every row chunk) on the launching stream
    t_step = scr_ms / max(1, steps)
    achieved = flops_per_step / (t_step * 1e-3) / 1e12 if scr_n else None
    peak = pk.get("bf16_tflops", pk.get("bf16_tflops_sustained"))
    peak_sus = pk.get("bf16_tflops_sustained")
    return {"bound": "tensor", "kernel": "screen_kernel (tcgen05 kind::f16, cta_group::2)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "peak_kind": f"{pk_kind} bf16 dense burst (f16 rate == bf16 rate)",
            "frac_vs_sustained": (achieved / peak_sus) if (achieved and peak_sus) else None,
            "algorithmic_flops_per_step": flops_per_step, "screen_ms_per_step": t_step}


def run_c2(torch, args, device):
    """BASELINE configs[1] (C2) on one GPU: N = 1,048,576 fp32 D=512 rows, K=1024,
    device-resident batch; plus its e2e through the public API with a pinned
    host batch (H2D inside the timed region) and the CPU port."""
    from paper_2603_09632_b200 import _native as nat
    from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
    import paper_2603_09632_b200 as xv
    cfg = xv.VqConfig(K=K, lam=LAM, gamma=0.5 / K, delta_dead=DELTA, epsilon=EPS, reservoir_capacity=CAP)
    x, E0 = make_data(torch, 0, device)
    be = CudaBackend(K, D, LAM, EPS)
    vq = DataParallelVQ((E0.clone(), torch.zeros(K, dtype=torch.float64, device=device),
                         torch.zeros(K, D, dtype=torch.float64, device=device)), cfg, np.random.default_rng(12), be)
    for _ in range(args.warmup):
        vq.step(x, [N_ROWS])
    steps = max(args.steps, 20)
    ms = timed_steps(torch, vq, x, [N_ROWS], steps, lambda: None, 1, device) / steps
    prof = profiled_steps(torch, vq, x, [N_ROWS], 10)
    cb_now = xv.Codebook._make(vq.state[0], vq.state[1], vq.state[2], LAM, EPS, None)
    _, (n_rerank, n_fallback) = xv.vq.assign_batch_stats(x, cb_now)
    xh = x.cpu().pin_memory()
    vq2 = DataParallelVQ((E0.clone(), torch.zeros(K, dtype=torch.float64, device=device),
                          torch.zeros(K, D, dtype=torch.float64, device=device)), cfg, np.random.default_rng(12), be)
    vq2.step(xh, [N_ROWS])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        vq2.step(xh, [N_ROWS])
        vq2.state[0].cpu()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / 3
    out = {"workload": WORKLOAD, "Mfeat_per_s": N_ROWS / (ms * 1e-3) / 1e6, "ms_per_step": ms, "steps": steps,
           "roofline": screen_roofline(prof, 2.0 * N_ROWS * K * D, 10, ncu_traffic("screen_kernel_C2")),
           "per_kernel": {t: {"ms_per_step": m / 10, "launches": c} for t, (m, c) in prof.items()},
           "assign_exact_rows": {"rerank": n_rerank, "fallback": n_fallback},
           "e2e": {"value": N_ROWS / (e2e_ms * 1e-3) / 1e6, "unit": "Mfeat/s", "h2d_bytes_per_step": N_ROWS * D * 4,
                   "d2h_bytes_per_step": K * D * 8, "ms_per_step": e2e_ms}}
    if not args.no_cpu:
        xs = x[:65536].cpu().numpy()
        v, thr, rows, el = cpu_port_rate(xs, E0.cpu().numpy(), seconds=args.cpu_seconds)
        out["cpu_baseline"] = {"value": v, "unit": "Mfeat/s", "cores": thr, "kind": "port",
                               "sample": f"{rows} rows of the C2 batch in {el:.1f}s (assign+accumulate, "
                                         f"oracle/oracle.c, {thr} threads)"}
    del x, xh, vq, vq2
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-grid", action="store_true")
    ap.add_argument("--no-c2", action="store_true")
    ap.add_argument("--grid-steps", type=int, default=5)
    ap.add_argument("--stream-frames", type=int, default=1000)
    args = ap.parse_args()
    # The timed regions must not see Python's cyclic-GC pauses (the CPU legs allocate
    # enough objects to trigger gen-2 collections in the middle of a later GPU
    # measurement: the rasterizer build read 33 ms instead of 1 ms): collect between
    # the sub-benchmarks instead.
    gc.collect()
    gc.disable()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        # NCCL's init lines (transport: NVLink / NVLS) go to stderr; the JSON line stays on stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH")
        dist.init_process_group("nccl", device_id=device)

    import paper_2603_09632_b200 as xv
    from paper_2603_09632_b200 import _native as nat
    from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------- headline: C5 strong scaling (67,108,864 rows split over the ranks)
    cfg = xv.VqConfig(K=C5_K, lam=LAM, gamma=0.5 / C5_K, delta_dead=DELTA, epsilon=EPS, reservoir_capacity=CAP)
    x, E0 = c5_data(torch, rank, world, device)
    rows = int(x.shape[0])
    from paper_2603_09632_b200.distributed import strong_shard
    sizes = [strong_shard(C5_TOTAL, world, r)[1] for r in range(world)]
    be = CudaBackend(C5_K, C5_D, LAM, EPS)
    state0 = (E0, torch.zeros(C5_K, dtype=torch.float64, device=device),
              torch.zeros(C5_K, C5_D, dtype=torch.float64, device=device))
    vq = DataParallelVQ(tuple(t.clone() for t in state0), cfg, np.random.default_rng(42), be)
    for _ in range(args.warmup):
        vq.step(x, sizes)
    clk = ClockSampler(local)
    clk.start()
    l0 = nat.launch_count()
    ms = timed_steps(torch, vq, x, sizes, args.steps, barrier, world, device)
    launches = nat.launch_count() - l0
    clocks = clk.stop()
    ms_step = ms / args.steps
    value = C5_TOTAL / (ms_step * 1e-3) / 1e6
    prof_steps = 3
    prof = profiled_steps(torch, vq, x, sizes, prof_steps)
    cb_now = xv.Codebook._make(vq.state[0], vq.state[1], vq.state[2], LAM, EPS, None)
    _, (n_rerank, n_fallback) = xv.vq.assign_batch_stats(x, cb_now)
    t5 = ncu_traffic("screen_kernel_C5_per_step")
    roof = screen_roofline(prof, 2.0 * rows * C5_K * C5_D, prof_steps,
                           t5 * rows / C5_TOTAL if t5 else None)
    roof["traffic_note"] = ("DRAM bytes per step of the screen kernel (all row-chunk launches) from the N=1 ncu "
                            "capture profiles/r2_c5_screen_pflate.csv, scaled by this rank's rows")

    # e2e through the public API: every step copies its rows from pinned host
    # memory (H2D inside the timed region, overlapped chunk by chunk with the
    # device work) and reads the updated codebook back.  Pinning the whole
    # 154.6 GB / N shard is not done: each step streams E2E_ROWS rows per rank
    # (the same distribution, K, D and dtype); the rate is PCIe-bound.
    del vq
    e2e_rows = min(min(sizes), (1 << 22) // world)   # ~9.7 GB of pinned host rows in total over the ranks
    xh = x[:e2e_rows].cpu().pin_memory()
    del x
    torch.cuda.empty_cache()
    vq2 = DataParallelVQ(tuple(t.clone() for t in state0), cfg, np.random.default_rng(42), be)
    e2e_sizes = [e2e_rows] * world
    vq2.step(xh, e2e_sizes)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(max(1, args.e2e_steps)):
        vq2.step(xh, e2e_sizes)
        vq2.state[0].cpu()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    e2e_ms = e0.elapsed_time(e1) / max(1, args.e2e_steps)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = world * e2e_rows / (e2e_ms * 1e-3) / 1e6
    del vq2, xh
    torch.cuda.empty_cache()

    cpu = c1 = c2 = grid = stream = targets = consumers = raster = init = None
    if rank == 0 and world == 1:
        def sub(fn, *a, **k):   # each sub-benchmark starts from a collected heap
            gc.collect()
            return fn(*a, **k)
        if not args.no_cpu:
            cpu = sub(cpu_port_c5, args.cpu_seconds)
        if not args.no_c2:
            c2 = sub(run_c2, torch, args, device)
        if not args.no_grid:
            c1 = sub(run_c1, torch, cpu=not args.no_cpu)
        # the C4 stream before the C3 grid: the per-device grid state (batch table)
        # would otherwise keep the size the 16-frame C3 batches gave it
        if args.stream_frames > 0:
            stream = sub(run_stream, torch, args.stream_frames, device)
        if not args.no_grid:
            grid = sub(run_grid, torch, args.grid_steps, cpu=not args.no_cpu)
        if not args.no_grid:
            targets = sub(run_targets, torch, 10, cpu=not args.no_cpu)
            init = sub(run_init, torch, cpu=not args.no_cpu)
            consumers = sub(run_consumers, torch, 5, cpu=not args.no_cpu)
            raster = sub(run_raster, torch, 7, cpu=not args.no_cpu)
    if rank == 0:
        per_kernel = {t: {"ms_per_step": m / prof_steps, "launches": c} for t, (m, c) in prof.items()}
        g1 = (grid or {}).get("0.01") or {}
        line = {
            "metric": "VQ Mfeat/s (online_step: assign + accumulate + EMA + revival), C5 strong scaling",
            "value": value, "unit": "Mfeat/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16 rows, f16-screen/f64-exact",
            "data": "synthetic (seeded 4096-centre unit-norm mixture, generated on device)",
            "config": {"workload": C5_WORKLOAD, "global_batch": C5_TOTAL, "rows_per_gpu": rows, "K": C5_K,
                       "D": C5_D, "parallelism": f"dp{world}", "iterations": args.steps,
                       "l2": "batch 154.6 GB / N per GPU > 126 MB L2 (no flush needed)"},
            "c5_ms_per_iter": ms_step, "c2_Mfeat_s": (c2 or {}).get("Mfeat_per_s"),
            "grid_c3_Gpts_s": (g1.get("Mpts_per_s") or 0) / 1e3 if g1 else None,
            "grid_c3_ms": g1.get("ms_per_batch"), "grid_front_hbm_frac": (g1.get("roofline") or {}).get("frac"),
            "grid_batch_hbm_frac": g1.get("batch_hbm_frac"),
            "grid_c3_graph_ms": (g1.get("graph") or {}).get("ms_per_batch"),
            "grid_front_issue_frac": ((g1.get("roofline") or {}).get("issue") or {}).get("frac"),
            "stream_p50_ms": (stream or {}).get("p50_ms"), "stream_p99_ms": (stream or {}).get("p99_ms"),
            "c1_ms": (c1 or {}).get("ms_per_frame_step"),
            "e2e": {"value": e2e_val, "unit": "Mfeat/s", "h2d_bytes_per_step": world * e2e_rows * C5_D * 2,
                    "d2h_bytes_per_step": C5_K * C5_D * 8, "ms_per_step": e2e_ms,
                    "rows_per_step": world * e2e_rows,
                    "note": "pinned host rows streamed into the step (H2D chunks overlapped with the device work); "
                            "4,194,304 / N rows per rank per step (the whole shard is not pinned), same K/D/dtype"},
            "gpu_launches": launches,
            "roofline": roof,
            "per_kernel": per_kernel,
            "assign_exact_rows": {"rerank": n_rerank, "fallback": n_fallback},
            "clocks": clocks,
            "cpu_baseline": cpu,
            "c1": c1,
            "c2": c2,
            "grid": grid,
            "stream": stream,
            "targets": targets,
            "consumers": consumers,
            "raster": raster,
            "init": init,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
